"""LSQR launch-list probe (development aid): c4, plain LSQR, a few iterations."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1602_06621_b200 as eq  # noqa: E402
from paper_1602_06621_b200 import configs  # noqa: E402

inst = configs.config(4)
b = configs.rhs(inst)
M = eq.ExplicitMatrix.from_csr(inst.m, inst.n, inst.row_ptr, inst.col, inst.val)
eq.lsqr(M, b, 2, 0.0)
r = eq.lsqr(M, b, int(sys.argv[1]) if len(sys.argv) > 1 else 10, 0.0)
print("ok", r.residual_history[-1])
