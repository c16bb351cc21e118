python -m pytest tests -m "gpu and not slow" -q 2>&1 | tail -5 > gpurun_out/t11.log
python tools/bench_extra.py multilinear > gpurun_out/extra11.jsonl 2> gpurun_out/extra11.err
tests/cpp/_build/bench_cpp 5 2 > gpurun_out/cpp11.json 2> gpurun_out/cpp11.err
