"""Handle-path step timeline on c3 (EQUIL_VERBOSE=2): signs / loop / finalize
phases of sgd_equilibrate on a resident matrix (development aid)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1602_06621_b200 as eq  # noqa: E402
from paper_1602_06621_b200 import configs  # noqa: E402

inst = configs.config(3)
M = eq.ExplicitMatrix.from_csr(inst.m, inst.n, inst.row_ptr, inst.col, inst.val)
p = eq.EquilibrationParams(alpha=inst.alpha, beta=inst.beta, iterations=100, seed=0)
for k in range(4):
    t0 = time.perf_counter()
    eq.sgd_equilibrate(M, p)
    print(f"step {1e3 * (time.perf_counter() - t0):.2f} ms", file=sys.stderr, flush=True)
