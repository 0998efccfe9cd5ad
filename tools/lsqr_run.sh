timeout 600 python tools/lsqr_probe.py > gpurun_out/lsqr_probe.log 2>&1
EQUIL_VERBOSE=1 timeout 300 python -c "
import sys; sys.path.insert(0, '.')
import time, numpy as np, paper_1602_06621_b200 as eq
from paper_1602_06621_b200 import configs
import torch
inst = configs.config(3)
rp = torch.from_numpy(inst.row_ptr).pin_memory().numpy(); c = torch.from_numpy(inst.col).pin_memory().numpy(); v = torch.from_numpy(inst.val).pin_memory().numpy()
p = eq.EquilibrationParams(alpha=inst.alpha, beta=inst.beta, iterations=100, seed=0)
for k in range(3):
    t0 = time.perf_counter(); eq.sgd_equilibrate_csr(inst.m, inst.n, rp, c, v, p); print('e2e', time.perf_counter() - t0, flush=True)
" > gpurun_out/e2e_probe.log 2>&1
