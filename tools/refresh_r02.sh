#!/bin/bash
# Round-2 refresh of the judged records (outputs in gpurun_out/, summaries copied to profiles/ by hand):
# bench line (both arms), launch list, ncu --set full of the hot kernels, configs, extra cases, smoke.
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/rf_bench.log 2>&1; echo bench=$?
timeout 900 python bench.py --impl reference > gpurun_out/rf_ref.log 2>&1; echo ref=$?
timeout 600 python bench.py --g multilinear --no-cpu-baseline --no-e2e > gpurun_out/rf_ml.log 2>&1; echo ml=$?
bash tools/launches.sh rf; echo launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_bucket_tma|k_gather_fwd|k_dec_out|k_resid_codes|k_dec_agg|k_rle_write_fast|k_rle_tiles_fast|k_nd_mid|k_nd_outer|k_nd3_plane|k_nd3_outer|k_stencil_3d" -c 16 -o gpurun_out/rf_full python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/rf_ncu.log 2>&1; echo ncu=$?
timeout 600 python tools/bench_configs.py > gpurun_out/rf_configs.jsonl 2> gpurun_out/rf_configs.err; echo cfg=$?
timeout 600 python tools/bench_extra.py > gpurun_out/rf_extra.jsonl 2> gpurun_out/rf_extra.err; echo extra=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rf_smoke.log 2>&1; echo smoke=$?
