#!/bin/bash
# usage: tools/ab_variants.sh v1 v2 ...   (A/B of variants/<v>/libumcg.so on the bench)
for v in base "$@"; do
  if [ "$v" == "base" ]; then unset UMCG_LIB_PATH; else export UMCG_LIB_PATH=$PWD/variants/$v/libumcg.so; fi
  python bench.py --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['compress']['ms'],3), round(d['decompress']['ms'],3), {k:round(v['ms'],3) for k,v in d['kernels'].items()})"
done
