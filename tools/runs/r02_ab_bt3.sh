python -m pytest tests/test_gpu_escapes.py -q -x -k "pipeline_outliers" 2>&1 | grep -E "Error|error|assert|passed|failed" | head -30 > gpurun_out/esc9.log
python -m pytest tests/test_gpu_parity.py tests/test_gpu_cpp.py -q 2>&1 | tail -5 >> gpurun_out/esc9.log
for v in 0 1; do UMCG_BT3=$v python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('BT3=$v', round(d['compress']['ms'],4), round(d['decompress']['ms'],4), {k:round(v['ms'],4) for k,v in d['kernels'].items()})" >> gpurun_out/ab9.log; done
UMCG_BT3=1 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2 >> gpurun_out/ab9.log
ncu --set full --clock-control none --import-source on -k regex:k_ml_bucket -s 1 -c 1 -o gpurun_out/r02_ml python tools/bench_extra.py multilinear > gpurun_out/ncu_ml.log 2>&1
