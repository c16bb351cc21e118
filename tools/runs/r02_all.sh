UMCG_PARITY_LOG=gpurun_out/fullsize4.jsonl timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -6 > gpurun_out/t16.log
bash tools/runs/r02_final.sh > gpurun_out/final16.log 2>&1
