#!/bin/bash
# usage: BENCH_CFG_ONLY=.. BENCH_CFG_QUICK=.. tools/ab_cfg.sh v1 v2 ... (tools/bench_configs.py per variant)
for v in base "$@"; do
  if [ "$v" == "base" ]; then unset UMCG_LIB_PATH; else export UMCG_LIB_PATH=$PWD/variants/$v/libumcg.so; fi
  timeout 600 python tools/bench_configs.py 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v', d['config'][:30], d['tau'], round(d['compress_ms'],3), round(d['decompress_ms'],3))"
done
