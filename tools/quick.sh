#!/bin/bash
# Quick GPU loop: optional non-slow GPU tests, a short bench and the compress /
# decompress phase traces. Usage: tools/quick.sh [tests] [tag]
mkdir -p gpurun_out
tag=${2:-q}
if [ "$1" = "tests" ]; then
  timeout 1200 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/${tag}_tests.log 2>&1
  echo "tests rc=$?" >> gpurun_out/${tag}_tests.log
fi
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_bench.log 2>&1
UMCG_COMP_TRACE=1 UMCG_DEC_TRACE=1 timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_trace.log 2>&1
python - "$tag" <<'PY'
import json, sys
tag = sys.argv[1]
l = [x for x in open(f'gpurun_out/{tag}_bench.log') if x.startswith('{')]
if l:
    d = json.loads(l[-1])
    print('compress', round(d['compress']['ms'], 4), 'decompress', round(d['decompress']['ms'], 4))
    print({k: round(v['ms'], 4) for k, v in d['kernels'].items()})
PY
grep "trace\]" gpurun_out/${tag}_trace.log | tail -16
