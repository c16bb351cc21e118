#!/bin/bash
# usage: tools/ab_e2e.sh v1 v2 ...   (A/B of variants/<v>/libumcg.so on the bench's e2e number)
for v in base "$@"; do
  if [ "$v" == "base" ]; then unset UMCG_LIB_PATH; else export UMCG_LIB_PATH=$PWD/variants/$v/libumcg.so; fi
  python bench.py --no-cpu-baseline 2>&1 | tail -1 | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('$v', round(e['value'],2), round(e['ms_per_step'],2), 'serial', round(e['serial']['value'],2), e['matches_device_path'])"
done
