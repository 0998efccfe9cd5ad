"""Per-phase times of one sgd_equilibrate call on a resident matrix (EQUIL_VERBOSE
phases synchronise; development aid) and the unsynchronised step time."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1602_06621_b200 as eq  # noqa: E402
from paper_1602_06621_b200 import configs  # noqa: E402

inst = configs.config(3)
M = eq.ExplicitMatrix.from_csr(inst.m, inst.n, inst.row_ptr, inst.col, inst.val)
p = eq.EquilibrationParams(alpha=inst.alpha, beta=inst.beta, iterations=100, seed=0)
bufs = [torch.empty(k, dtype=torch.float64, device="cuda") for k in (inst.m, inst.n, inst.m, inst.n)]
for k in range(int(os.environ.get("STEPS", "4"))):
    t0 = time.perf_counter()
    eq.sgd_equilibrate_device(M, p, *[b.data_ptr() for b in bufs])
    t1 = time.perf_counter()
    ms, it = eq.last_loop_ms(M)
    print(f"step {1e3 * (t1 - t0):.2f} ms  loop {ms:.2f} ms", file=sys.stderr, flush=True)
