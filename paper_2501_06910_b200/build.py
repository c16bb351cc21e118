"""Build libumcg.so (the sm_100a product library) in-tree with nvcc.

Every translation unit is compiled for sm_100a only, with --fmad=false so no
floating-point contraction happens anywhere on the path (the reference is
built with -ffp-contract=off, proj/CMakeLists.txt:16-17), and -lineinfo so
ncu's source page maps to these files.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libumcg.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + ["-O3", "-lineinfo", "--fmad=false", "-std=c++17", "-Xcompiler", "-fPIC",
                "-Xcompiler", "-O3", "-Xcompiler", "-fopenmp", "--expt-relaxed-constexpr", "-Xptxas", "-v"]

SOURCES = ["encode.cu", "partition.cu", "stream.cu", "codes.cu", "decode.cu", "interp.cu", "plan.cu", "api.cu", "datagen.cu", "gridinit.cu", "escape.cu", "digest.cu", "radix.cu"]


def _needs(src: str, obj: str) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    deps = [src] + [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".h", ".cuh"))]
    deps.append(os.path.join(HERE, "..", "include", "umcg.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(name: str, verbose: bool) -> str:
    src = os.path.join(CSRC, name)
    obj = os.path.join(BUILD, name.replace(".cu", ".o"))
    if not _needs(src, obj):
        return ""
    cmd = [NVCC] + FLAGS + ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {name}:\n{r.stderr}")
    log = r.stderr
    with open(obj + ".ptxas.log", "w") as f:
        f.write(log)
    return f"[{name}] compiled" + ("\n" + log if verbose else "")


def _flags_changed() -> bool:
    """Objects are rebuilt whenever the compile flags change (mtimes alone
    would keep objects built with different flags)."""
    stamp = os.path.join(BUILD, "flags.txt")
    want = " ".join(FLAGS)
    have = open(stamp).read() if os.path.exists(stamp) else ""
    if have != want:
        for f in os.listdir(BUILD):
            if f.endswith(".o"):
                os.remove(os.path.join(BUILD, f))
        with open(stamp, "w") as fh:
            fh.write(want)
        return True
    return False


def build(verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    _flags_changed()
    with cf.ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 4)) as ex:
        outs = list(ex.map(lambda s: _compile(s, verbose), SOURCES))
    objs = [os.path.join(BUILD, s.replace(".cu", ".o")) for s in SOURCES]
    if not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart", "-lgomp"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
        outs.append(f"linked {LIB}")
    return "\n".join(o for o in outs if o)


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
