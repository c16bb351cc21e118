#!/bin/bash
# usage: tools/ab_env.sh VAR v1 v2 ...   (A/B of an environment knob on the bench)
var=$1; shift
for v in "$@"; do
  env $var=$v python bench.py --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$var=$v', round(d['compress']['ms'],3), round(d['decompress']['ms'],3), {k:round(v['ms'],3) for k,v in d['kernels'].items()})"
done
