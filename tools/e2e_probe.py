"""e2e phase probe (development aid): create / sgd / destroy times of the
one-shot path from pinned host CSR, c3."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1602_06621_b200 as eq  # noqa: E402
from paper_1602_06621_b200 import configs  # noqa: E402

inst = configs.config(3)
rp = torch.from_numpy(inst.row_ptr).pin_memory().numpy()
c = torch.from_numpy(inst.col).pin_memory().numpy()
v = torch.from_numpy(inst.val).pin_memory().numpy()
p = eq.EquilibrationParams(alpha=inst.alpha, beta=inst.beta, iterations=100, seed=0)
for k in range(4):
    t0 = time.perf_counter()
    M = eq.ExplicitMatrix.from_csr(inst.m, inst.n, rp, c, v)
    t1 = time.perf_counter()
    r = eq.sgd_equilibrate(M, p)
    t2 = time.perf_counter()
    M.close()
    t3 = time.perf_counter()
    t4 = time.perf_counter()
    eq.sgd_equilibrate_csr(inst.m, inst.n, rp, c, v, p)
    t5 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.1f} ms  sgd {1e3*(t2-t1):.1f} ms  destroy {1e3*(t3-t2):.1f} ms  "
          f"one-shot {1e3*(t5-t4):.1f} ms", flush=True)
