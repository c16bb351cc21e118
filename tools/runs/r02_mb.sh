./tools/mb_scatter2 > gpurun_out/mb_scatter2.log 2>&1
tests/cpp/_build/bench_cpp 5 2 > gpurun_out/cpp13.json 2> gpurun_out/cpp13.err
UMCG_DEC_TRACE=1 python -c "
import sys; sys.path.insert(0,'.')
import numpy as np, torch, paper_2501_06910_b200 as umcg
xyz, x = umcg.gen_config(3, 512, 0x250106910 + 3, device='cuda')
plan = umcg.Plan.build([np.linspace(0.0, 1.0, 256) for _ in range(3)], xyz)
b = umcg.Budget(tau=1e-4)
ar = torch.empty(plan.compress_bound('f'), dtype=torch.uint8, device='cuda')
out = torch.empty(plan.n, dtype=torch.float64, device='cuda')
L = plan.compress_into(x, b, ar, 'f')
for _ in range(4): plan.decompress_into(ar, L, out)
torch.cuda.synchronize()
" > gpurun_out/dectrace.log 2>&1
