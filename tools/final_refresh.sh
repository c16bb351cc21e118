mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_final.log 2>&1; echo bench=$?
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_final.log 2>&1; echo ref=$?
bash tools/launches.sh r01z; echo launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_bucket_tma|k_gather_fwd|k_dec_out|k_resid_codes|k_dec_agg|k_rle_write_fast|k_nd_mid|k_nd_outer" -c 12 -o gpurun_out/r01z_full python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_z.log 2>&1; echo ncu=$?
timeout 600 python tools/bench_configs.py > gpurun_out/configs_z.jsonl 2>gpurun_out/configs_z.err; echo cfg=$?
