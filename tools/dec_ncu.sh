# GPU loop for the decompress chain: tests, quick bench + traces, ncu launch
# list of config-3 decompress with the 3-D grid path on and off.
mkdir -p gpurun_out
tag=${1:-dec}
timeout 600 python -m pytest tests/test_gpu_nd3.py -x -q > gpurun_out/${tag}_nd3tests.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_nd3tests.log
bash tools/quick.sh tests $tag
for v in on off; do
  if [ $v = off ]; then export UMCG_ND3_OFF=1; fi
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_dec|k_nd|k_scan|k_tok|k_fast" --csv --log-file gpurun_out/${tag}_launches_$v.csv python tools/dec_only.py 2 > gpurun_out/${tag}_ncu_$v.log 2>&1
done
