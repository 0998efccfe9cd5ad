"""Setup/e2e phase timing (development aid): EQUIL_VERBOSE=1 python tools/e2e_probe.py [cfg]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1602_06621_b200 as eq  # noqa: E402
from paper_1602_06621_b200 import configs  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 3
inst = configs.config(k)
rp = torch.from_numpy(inst.row_ptr).pin_memory().numpy()
c = torch.from_numpy(inst.col).pin_memory().numpy()
v = torch.from_numpy(inst.val).pin_memory().numpy()
p = eq.EquilibrationParams(alpha=inst.alpha, beta=inst.beta, iterations=inst.iterations,
                           seed=inst.seed)
for rep in range(3):
    t0 = time.perf_counter()
    M = eq.ExplicitMatrix.from_csr(inst.m, inst.n, rp, c, v)
    t1 = time.perf_counter()
    r = eq.sgd_equilibrate(M, p)
    t2 = time.perf_counter()
    M.close()
    t3 = time.perf_counter()
    print(f"create {1e3 * (t1 - t0):.1f} ms  sgd {1e3 * (t2 - t1):.1f} ms  destroy "
          f"{1e3 * (t3 - t2):.1f} ms", flush=True)
    t0 = time.perf_counter()
    eq.sgd_equilibrate_csr(inst.m, inst.n, rp, c, v, p)
    print(f"one-shot e2e {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
