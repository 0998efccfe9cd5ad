"""LSQR iterations on c4 for an ncu launch list (development aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1602_06621_b200 as eq  # noqa: E402
from paper_1602_06621_b200 import configs  # noqa: E402

c4 = configs.config(4)
b = configs.rhs(c4)
M = eq.ExplicitMatrix.from_csr(c4.m, c4.n, c4.row_ptr, c4.col, c4.val)
eq.lsqr(M, b, 2, 0.0)
eq.lsqr(M, b, 10, 0.0)
print("ok")
