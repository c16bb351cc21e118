python -m pytest tests/test_gpu_escapes.py tests/test_gpu_parity.py -q -k "escape or outlier or wavefront or lossless or nd_" 2>&1 | tail -3 > gpurun_out/t17.log
python tools/bench_extra.py escape > gpurun_out/esc17_coop.jsonl 2>&1
UMCG_WAVE_LAUNCHES=1 python tools/bench_extra.py escape > gpurun_out/esc17_launch.jsonl 2>&1
