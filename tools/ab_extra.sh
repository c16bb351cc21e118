#!/bin/bash
# usage: tools/ab_extra.sh v1 v2 ...  (tools/bench_extra.py cases for base and variants/<v>/libumcg.so)
for v in base "$@"; do
  if [ "$v" == "base" ]; then unset UMCG_LIB_PATH; else export UMCG_LIB_PATH=$PWD/variants/$v/libumcg.so; fi
  timeout 400 python tools/bench_extra.py 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v', d['case'][:40], round(d['compress_ms'],3), round(d['decompress_ms'],3), {k:round(x,3) for k,x in d['kernels_ms'].items() if k in ('k_ml_resid','k_ml_recompose','k_resid_codes')})"
done
