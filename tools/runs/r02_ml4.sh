python -m pytest tests -m "gpu and not slow" -q -x 2>&1 | tail -3 > gpurun_out/t14.log
UMCG_PARITY_LOG=gpurun_out/ml14.jsonl python -m pytest tests/test_gpu_fullsize.py -q -k "multilinear" 2>&1 | tail -2 >> gpurun_out/t14.log
for v in base mlu4b3 mlu2b4 mlu8b3; do
  if [ "$v" == "base" ]; then unset UMCG_LIB_PATH; else export UMCG_LIB_PATH=$PWD/variants/$v/libumcg.so; fi
  echo "== $v" >> gpurun_out/ml14.log
  python tools/bench_extra.py multilinear 2>&1 | tail -1 >> gpurun_out/ml14.log
done
unset UMCG_LIB_PATH
