bash tools/ab_variants.sh btsum > gpurun_out/ab_btsum.log 2>&1
bash tools/ab_variants.sh btsum >> gpurun_out/ab_btsum.log 2>&1
