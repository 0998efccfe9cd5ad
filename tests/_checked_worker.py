"""Workload of tests/test_gpu_checked.py (the checked build, EQ_CHECK asserts)
and tests/test_gpu_sanitizer.py (compute-sanitizer, where the pool allows it).

    EQUIL_LIB=paper_1602_06621_b200/libequil_b200_checked.so python tests/_checked_worker.py CASE

CASE c1: config 1 (10000 x 5000), SGD with history, plain and preconditioned
LSQR, apply / adjoint.  CASE c3s: config 3 at 5% (100000 x 50000, Zipf rows up
to 10^4 entries, so the warp-specialised long-slice kernel and its mbarrier
ring run), SGD with the RMS / objective history over m + n >= 1e5 terms, and
LSQR.  CASE blocks: forced column-block rounds (the carries between rounds).
Exits non-zero if a result differs from the oracle, so a sanitizer-clean run
is also a correct one.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402  (checker)
import paper_1602_06621_b200 as eq  # noqa: E402
from paper_1602_06621_b200 import configs  # noqa: E402


def main(case):
    inst = configs.config(1) if case == "c1" else configs.config(3, scale=0.05)
    A = oracle.CsrArrays(inst.m, inst.n, inst.row_ptr, inst.col, inst.val)
    C = oracle.c_oracle()
    M = eq.ExplicitMatrix.from_csr(inst.m, inst.n, inst.row_ptr, inst.col, inst.val)
    T = 4
    r = eq.sgd_equilibrate(M, eq.EquilibrationParams(iterations=T, seed=3),
                           eq.DiagnosticsConfig(stride=2))
    w = C.sgd_equilibrate(A, iterations=T, seed=3, diag_stride=2)
    for k in "uvde":
        assert np.array_equal(getattr(r, k), getattr(w, k)), k
    np.testing.assert_allclose([h.rms for h in r.history], w.hist_rms, rtol=1e-9)
    b = np.random.default_rng(1).standard_normal(inst.m)
    lp = eq.lsqr(M, b, 4, 0.0)
    assert np.array_equal(lp.residual_history, C.lsqr(A, b, 4, 0.0).residual_history)
    pp = eq.lsqr_preconditioned(M, b, eq.EquilibrationParams(iterations=2, seed=1), 3, 0.0)
    assert np.array_equal(pp.residual_history,
                          C.lsqr_preconditioned(A, b, 3, 0.0, iterations=2, seed=1).residual_history)
    x = np.random.default_rng(2).standard_normal(inst.n)
    assert np.array_equal(M.apply(x), C.apply(A, x))
    print("ok", case, "build_flags", eq._lib.load().equil_build_flags(), flush=True)


if __name__ == "__main__":
    main(sys.argv[1])
