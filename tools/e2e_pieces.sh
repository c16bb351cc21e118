#!/bin/bash
# e2e HostPipeline step time against the piece size of the pinned host copies (UMCG_PIECE_MB)
for mb in 8 32 64 256 4096; do
  echo "piece ${mb} MiB"; UMCG_PIECE_MB=$mb timeout 600 python tools/e2e_timeline.py 2>&1 | grep "concurrent\|2c/2d plans k=16"
done
