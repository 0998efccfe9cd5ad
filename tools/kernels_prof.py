"""Drive every hot kernel once for an ncu capture (development aid): dense c2
SGD iterations, c4 LSQR iterations (pass_kernel, reductions), c3 setup
(transpose, validation, slots, sign stream)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1602_06621_b200 as eq  # noqa: E402
from paper_1602_06621_b200 import configs  # noqa: E402

c2 = configs.config(2)
D = eq.ExplicitMatrix.dense(c2.dense)
eq.sgd_equilibrate(D, eq.EquilibrationParams(alpha=c2.alpha, beta=c2.beta, iterations=3, seed=1))
del D
c4 = configs.config(4)
b = configs.rhs(c4)
M = eq.ExplicitMatrix.from_csr(c4.m, c4.n, c4.row_ptr, c4.col, c4.val)
eq.lsqr(M, b, 3, 0.0)
eq.sgd_equilibrate(M, eq.EquilibrationParams(iterations=3))
print("ok")
