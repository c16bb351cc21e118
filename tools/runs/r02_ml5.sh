for v in mlu2b4 mlu2b5 mlu2b6 mlu1b6 mlu3b4; do
  export UMCG_LIB_PATH=$PWD/variants/$v/libumcg.so
  echo "== $v" >> gpurun_out/ml15.log
  python tools/bench_extra.py multilinear 2>&1 | tail -1 >> gpurun_out/ml15.log
done
