"""The matrix-free entry point (equil_sgd_equilibrate_operator): projected-SGD
equilibration of a LinearOperator given only by device apply / apply_adjoint
callbacks (include/equil/linop.hpp:13-25; sgd_equilibrate,
src/equilibrate.cpp:138-221).  With an explicit matrix's own device apply as
the operator, the result must equal the explicit path and the oracle bit for
bit; a purely matrix-free operator (the identity as a device copy) must stay
at the fixed point (tests/test_equilibrate.cpp:183-198)."""
import ctypes
import os

import numpy as np
import pytest

import oracle
import paper_1602_06621_b200 as eq
from conftest import csr_from_golden

pytestmark = pytest.mark.gpu


def _matrix(A):
    if A.dense is not None:
        return eq.ExplicitMatrix.dense(A.dense)
    return eq.ExplicitMatrix.from_csr(A.m, A.n, A.row_ptr, A.col, A.val)


@pytest.mark.parametrize("case", ["sp", "lr", "dn", "c3"])
def test_operator_path_bit_exact(C, golden, case):
    if case == "c3":
        from paper_1602_06621_b200 import configs
        inst = configs.config(3, scale=0.02)
        A = oracle.CsrArrays(inst.m, inst.n, inst.row_ptr, inst.col, inst.val)
    else:
        A = csr_from_golden(golden, case)
    M = _matrix(A)
    p = eq.EquilibrationParams(iterations=30, seed=5)
    want = eq.sgd_equilibrate(M, p)
    got = eq.sgd_equilibrate_operator(eq.DeviceOperator.from_matrix(M), p)
    for k in "uvde":
        assert np.array_equal(getattr(got, k), getattr(want, k)), k
    assert (got.box_feasible, got.iterate_bound_ok) == (want.box_feasible, want.iterate_bound_ok)
    assert (got.apply_count, got.adjoint_count) == (30, 30)
    assert (got.alpha, got.beta) == (want.alpha, want.beta)
    w = C.sgd_equilibrate(A, iterations=30, seed=5)
    for k in "uvde":
        assert np.array_equal(getattr(got, k), getattr(w, k)), ("oracle", k)


def _cudart():
    for name in ("libcudart.so.12", "/usr/local/cuda/lib64/libcudart.so.12"):
        try:
            return ctypes.CDLL(name)
        except OSError:
            continue
    pytest.skip("libcudart not found")


def test_matrix_free_identity_stays_at_fixed_point():
    rt = _cudart()
    rt.cudaMemcpyAsync.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                   ctypes.c_int, ctypes.c_void_p]
    n = 9
    calls = []

    def copy(i, o, s):  # y = x on the device, on our stream
        calls.append(1)
        assert rt.cudaMemcpyAsync(o, i, n * 8, 3, s) == 0

    op = eq.DeviceOperator(n, n, copy, copy)
    r = eq.sgd_equilibrate_operator(op, eq.EquilibrationParams(alpha=1.0, beta=1.0,
                                                               iterations=25))
    assert len(calls) == 50
    assert np.all(r.u == 0) and np.all(r.v == 0) and np.all(r.d == 1) and np.all(r.e == 1)
    assert r.box_feasible and r.iterate_bound_ok


def test_operator_parameter_errors_match_the_reference_messages():
    op = eq.DeviceOperator(3, 2, lambda i, o, s: None, lambda i, o, s: None)
    with pytest.raises(eq.InvalidArgument, match="gamma must be positive"):
        eq.sgd_equilibrate_operator(op, eq.EquilibrationParams(gamma=0.0))
    with pytest.raises(eq.InvalidArgument, match="m\\*alpha\\^2 == n\\*beta\\^2"):
        eq.sgd_equilibrate_operator(op, eq.EquilibrationParams(alpha=1.0, beta=1.0))
    r = eq.sgd_equilibrate_operator(op, eq.EquilibrationParams(iterations=0))
    assert np.all(r.u == 0) and np.all(r.d == 1) and r.apply_count == 0


@pytest.mark.parametrize("case", ["sp", "lr", "dn"])
def test_operator_lsqr_bit_exact(golden, case):
    """lsqr / lsqr_preconditioned on the operator (src/lsqr.cpp:17-138 step by
    step: three operator calls per iteration) equal the explicit path, which
    is pinned to the reference's golden runs."""
    A = csr_from_golden(golden, case)
    M = _matrix(A)
    op = eq.DeviceOperator.from_matrix(M)
    b = np.random.default_rng(11).standard_normal(A.m)
    got = eq.lsqr_operator(op, b, 25, 0.0)
    want = eq.lsqr(M, b, 25, 0.0)
    assert np.array_equal(got.x, want.x)
    assert got.residual_history == want.residual_history
    assert (got.iterations, got.breakdown, got.reached_tol) == \
        (want.iterations, want.breakdown, want.reached_tol)
    assert (got.apply_count, got.adjoint_count) == (want.apply_count, want.adjoint_count)
    p = eq.EquilibrationParams(iterations=15, seed=3)
    got = eq.lsqr_operator(op, b, 25, 0.0, p)
    want = eq.lsqr_preconditioned(M, b, p, 25, 0.0)
    assert np.array_equal(got.x, want.x)
    assert got.residual_history == want.residual_history
    assert (got.iterations, got.equil_iterations) == (want.iterations, want.equil_iterations)
    assert (got.apply_count, got.adjoint_count) == (want.apply_count, want.adjoint_count)


def test_operator_lsqr_errors_and_breakdown():
    rt = _cudart()
    rt.cudaMemcpyAsync.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                   ctypes.c_int, ctypes.c_void_p]
    rt.cudaMemsetAsync.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t,
                                   ctypes.c_void_p]
    n = 6
    ident = eq.DeviceOperator(n, n, lambda i, o, s: rt.cudaMemcpyAsync(o, i, n * 8, 3, s),
                              lambda i, o, s: rt.cudaMemcpyAsync(o, i, n * 8, 3, s))
    b = np.arange(1.0, n + 1)
    r = eq.lsqr_operator(ident, b, 10, 1e-12)  # test_itersolvers.cpp:36-46
    assert r.reached_tol and r.iterations == 1 and r.residual_history[0] == 1.0
    assert np.allclose(r.x, b)
    with pytest.raises(eq.InvalidArgument, match="rhs must be nonzero"):
        eq.lsqr_operator(ident, np.zeros(n), 5, 0.0)
    with pytest.raises(eq.InvalidArgument, match="max_iters must be nonnegative"):
        eq.lsqr_operator(ident, b, -1, 0.0)
    zero = eq.DeviceOperator(n, n, lambda i, o, s: rt.cudaMemsetAsync(o, 0, n * 8, s),
                             lambda i, o, s: rt.cudaMemsetAsync(o, 0, n * 8, s))
    r = eq.lsqr_operator(zero, b, 10, 0.0)  # A^T b = 0: breakdown at setup
    assert r.breakdown and r.iterations == 0 and np.all(r.x == 0)
