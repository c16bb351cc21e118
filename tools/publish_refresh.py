"""Copy the outputs of tools/refresh_r02.sh (gpurun_out/rf_*) into profiles/:
bench lines, launch list, ncu table + per-kernel DRAM traffic, configs, extra
cases, smoke log. Usage: python tools/publish_refresh.py [round_tag]"""
import os
import shutil
import subprocess
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, P = os.path.join(R, "gpurun_out"), os.path.join(R, "profiles")


def last_json(src, dst):
    lines = [x for x in open(os.path.join(G, src)) if x.startswith("{")]
    if not lines:
        sys.exit(f"{src}: no JSON line")
    open(os.path.join(P, dst), "w").write(lines[-1])


last_json("rf_bench.log", f"{tag}_bench_full.json")
last_json("rf_ref.log", f"{tag}_bench_reference.json")
last_json("rf_ml.log", f"{tag}_bench_multilinear.json")
for src, dst in (("launches_rf.csv", f"{tag}_launches.csv"), ("rf_configs.jsonl", f"{tag}_configs.jsonl"),
                 ("rf_extra.jsonl", f"{tag}_extra.jsonl"), ("rf_smoke.log", f"{tag}_smoke.log")):
    shutil.copy(os.path.join(G, src), os.path.join(P, dst))
ll = subprocess.run([sys.executable, os.path.join(R, "tools", "summarize_launches.py"),
                     os.path.join(G, "launches_rf.csv"), "40"], capture_output=True, text=True).stdout
md = os.path.join(P, f"{tag}_launches.md")
head = open(md).read().split("```")[0] if os.path.exists(md) else f"# {tag} launch list\n\n"
open(md, "w").write(head + "```\n" + ll + "```\n")
tmp_md, traffic = os.path.join(G, "ncu_table.md"), os.path.join(P, "ncu_traffic.json")
subprocess.run([sys.executable, os.path.join(R, "tools", "ncu_table.py"), os.path.join(G, "rf_full.ncu-rep"), tmp_md,
                traffic], check=True, capture_output=True)
summ = os.path.join(P, f"{tag}_ncu_full_summary.md")
head = open(summ).read().split("| kernel |")[0] if os.path.exists(summ) else f"# {tag} ncu --set full summary\n\n"
open(summ, "w").write(head + open(tmp_md).read())
print("published", tag)
