"""CPU: the C-ABI library loads and exports every symbol include/umcg.h
declares (no compute calls: there is no GPU here)."""
import os
import re

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "umcg.h")).read()
    return sorted(set(re.findall(r"\b(umcg_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_the_python_export_list():
    import paper_2501_06910_b200 as u
    assert sorted(u.EXPORTED) == header_symbols()


def test_library_exports_every_declared_symbol():
    import paper_2501_06910_b200 as u
    L = u.lib()
    for sym in header_symbols():
        assert hasattr(L, sym), sym
    assert b"sm_100a" in L.umcg_version()


def test_library_is_sm100a_only():
    import subprocess
    so = os.path.join(ROOT, "paper_2501_06910_b200", "libumcg.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    arches = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert arches == {"100a"}, arches


def test_status_numbering_follows_reference_taxonomy():
    text = open(os.path.join(ROOT, "include", "umcg.h")).read()
    order = ["ERROR", "MALFORMED_FILE", "INDEX_OUT_OF_RANGE", "NON_FINITE_VALUE", "IO_FAILURE",
             "DEGENERATE_MESH", "EMPTY_AFTER_FILTERING", "INTERNAL_INCONSISTENCY",
             "SEED_MODE_UNSUPPORTED", "UNKNOWN_CODEC", "CORRUPT_PAYLOAD", "EXTERNAL_CODEC_VIOLATION",
             "SUBPROCESS_FAILURE", "BUDGET_INADMISSIBLE", "MAPPING_MISMATCH", "ZERO_NORM_REFERENCE",
             "MISMATCHED_RUNS"]
    for i, name in enumerate(order, start=1):
        assert re.search(rf"UMCG_{name} = {i},", text), name


def test_no_cpu_fallback_without_library(tmp_path, monkeypatch):
    import importlib
    import paper_2501_06910_b200 as u
    monkeypatch.setattr(u, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(u, "_lib", None)
    with pytest.raises(ImportError):
        u.lib()
    importlib.reload(u)
