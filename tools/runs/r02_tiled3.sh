python -m pytest tests/test_gpu_escapes.py tests/test_gpu_parity.py -q -k "escape or outlier or wavefront or lossless or nd_ or codec" 2>&1 | tail -2 > gpurun_out/t23.log
python tools/bench_extra.py escape 2>&1 | tail -1 > gpurun_out/esc23.jsonl
