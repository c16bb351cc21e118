python -m pytest tests/test_gpu_escapes.py -q -k "seed_mode or positions" 2>&1 | tail -2 > gpurun_out/t25.log
UMCG_COMP_TRACE=1 python -c "
import sys; sys.path.insert(0,'.')
import numpy as np, torch, paper_2501_06910_b200 as umcg
xyz, x = umcg.gen_config(3, 512, 0x250106910 + 3, device='cuda')
plan = umcg.Plan.build([np.linspace(0.0, 1.0, 256) for _ in range(3)], xyz)
b = umcg.Budget(tau=1e-4)
ar = torch.empty(plan.compress_bound('f'), dtype=torch.uint8, device='cuda')
for _ in range(4): plan.compress_into(x, b, ar, 'f')
torch.cuda.synchronize()
" > gpurun_out/comptrace25.log 2>&1
