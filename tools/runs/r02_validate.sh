timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -6 > gpurun_out/t24.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke24.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke24.log
