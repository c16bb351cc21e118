python -m pytest tests -m "gpu and not slow" -q 2>&1 | tail -3 > gpurun_out/t22.log
python -m pytest tests/test_gpu_fullsize.py -q -k "multilinear" 2>&1 | tail -2 >> gpurun_out/t22.log
python tools/bench_extra.py escape 2>&1 | tail -1 > gpurun_out/esc22.jsonl
python tools/bench_extra.py multilinear 2>&1 | tail -1 > gpurun_out/ml22.jsonl
