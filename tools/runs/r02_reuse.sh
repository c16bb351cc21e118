python -m pytest tests/test_gpu_escapes.py tests/test_gpu_fuzz.py tests/test_gpu_parity.py -q 2>&1 | tail -3 > gpurun_out/t32.log
python tools/bench_extra.py escape 2>&1 | tail -1 > gpurun_out/esc32.jsonl
UMCG_NO_REUSE=1 python tools/bench_extra.py escape 2>&1 | tail -1 > gpurun_out/esc32_noreuse.jsonl
