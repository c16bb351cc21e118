#!/bin/bash
# usage: tools_launches.sh <tag> [bench args...]; launch list of one bench step under ncu
tag=$1; shift
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e "$@" > gpurun_out/plain_$tag.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_$tag.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e "$@" > gpurun_out/ncu_$tag.log 2>&1
echo "launches rc=$?"
