#!/bin/bash
# Full-size single-core CPU reference measurement:
# config 3 at 512^3 / 256^3, tau_rel 1e-4, host-generated inputs, the
# reference's grid_coarsen, median of 3 round trips pinned to one CPU, the
# mapping_digest time for the "minus digest" figure. Run on the GPU box's host:
#   gpurun -- 'bash tools/cpu_full.sh gpurun_out/r02_cpu_full.json'
set -e
out=${1:-profiles/r02_cpu_full.json}
pin=$(python -c 'import os; print(sorted(os.sched_getaffinity(0))[-1])')
python -m oracle.cpu_bench --block 512 --reps 3 --tau 1e-4 --pin "$pin" > "$out"
cat "$out"
