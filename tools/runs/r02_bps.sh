for b in 1 2 4 8; do UMCG_WAVE_BPS=$b python tools/bench_extra.py escape 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('bps=$b', round(d['compress_ms'],2), round(d['decompress_ms'],2), {k:round(v,2) for k,v in d['kernels_ms'].items() if 'esc' in k})" >> gpurun_out/bps19.log; done
