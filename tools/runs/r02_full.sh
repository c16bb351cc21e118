cat /sys/kernel/mm/transparent_hugepage/enabled > gpurun_out/thp.txt 2>&1
rm -f gpurun_out/fullsize3.jsonl
UMCG_PARITY_LOG=gpurun_out/fullsize3.jsonl timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -8 > gpurun_out/t12.log
timeout 900 python tools/bench_configs.py > gpurun_out/configs12.jsonl 2> gpurun_out/configs12.err
timeout 600 python tools/bench_extra.py escape > gpurun_out/extra12.jsonl 2> gpurun_out/extra12.err
tests/cpp/_build/bench_cpp 5 2 > gpurun_out/cpp12.json 2> gpurun_out/cpp12.err
