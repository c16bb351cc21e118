python -m pytest tests/test_gpu_escapes.py tests/test_gpu_parity.py tests/test_gpu_cpp.py -q 2>&1 | tail -5 > gpurun_out/t10.log
python tools/bench_extra.py multilinear > gpurun_out/extra10.jsonl 2> gpurun_out/extra10.err
tests/cpp/_build/bench_cpp 5 2 > gpurun_out/cpp10.json 2> gpurun_out/cpp10.err
ncu --set full --clock-control none --import-source on -k regex:k_ml_bucket -s 1 -c 1 -o gpurun_out/r02_ml2 python tools/bench_extra.py multilinear > gpurun_out/ncu_ml2.log 2>&1
