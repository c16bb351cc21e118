#!/bin/bash
# Round-2 final measurement refresh (run on the GPU box after the tests pass):
# bench line (both arms), launch list, ncu --set full table of the hot kernels
# (nearest and multilinear), configs.
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo bench=$?
timeout 900 python bench.py --impl reference > gpurun_out/r02_bench_ref.json 2> gpurun_out/r02_bench_ref.err; echo ref=$?
timeout 600 python bench.py --g multilinear --no-cpu-baseline --no-e2e > gpurun_out/r02_bench_ml.json 2> gpurun_out/r02_bench_ml.err; echo ml=$?
bash tools/launches.sh r02; echo launches=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:k_bucket_tma|k_gather_fwd|k_dec_out|k_resid_codes|k_dec_agg|k_rle_write_fast|k_nd_mid|k_nd_outer" -c 12 -o gpurun_out/r02_full python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_r02_full.log 2>&1; echo ncu=$?
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_ml_bucket|k_add_gathered" -c 3 -o gpurun_out/r02_ml_full python bench.py --g multilinear --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_r02_ml.log 2>&1; echo ncu_ml=$?
