"""LSQR timing probe on c4 (development aid): wall time of lsqr / lsqr_preconditioned
at several iteration counts, and the e2e phase breakdown of the one-shot CSR call."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1602_06621_b200 as eq  # noqa: E402
from paper_1602_06621_b200 import configs  # noqa: E402

inst = configs.config(4)
b = configs.rhs(inst)
M = eq.ExplicitMatrix.from_csr(inst.m, inst.n, inst.row_ptr, inst.col, inst.val)
p = eq.EquilibrationParams(iterations=50)
for name, fn in [("lsqr", lambda k: eq.lsqr(M, b, k, 0.0)),
                 ("lsqr_pre", lambda k: eq.lsqr_preconditioned(M, b, p, k, 0.0))]:
    fn(3)
    for k in [0, 10, 60, 110, 110]:
        t0 = time.perf_counter()
        r = fn(k)
        dt = time.perf_counter() - t0
        print(name, k, f"{dt * 1e3:.2f} ms", r.iterations, len(r.residual_history),
              r.residual_history[-1], flush=True)
