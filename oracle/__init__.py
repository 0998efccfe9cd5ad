"""ctypes bindings for the parity checkers (TEST INFRASTRUCTURE).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs import this package.  The product
(paper_1602_06621_b200) never does.

Two checkers:
  * ``C``   -- liboracle.so, the plain-C restatement (equil_oracle.c);
  * ``Ref`` -- _ref/libequil_ref.so, the reference's own sources compiled
               unmodified against eigen_lite (built here from /root/reference;
               the prebuilt .so travels to the GPU box).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libequil_ref.so")
REFERENCE_SRC = "/root/reference/proj"

_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)
_u32p = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)
_ip = C.POINTER(C.c_int)


def build(ref: bool = True) -> None:
    """Compile liboracle.so (and _ref when the reference sources exist)."""
    targets = ["all"]
    if ref and os.path.isdir(REFERENCE_SRC):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


def ptr(a: np.ndarray | None, t):
    if a is None:
        return C.cast(None, t)
    assert a.flags.c_contiguous
    return a.ctypes.data_as(t)


class _Params(C.Structure):
    _fields_ = [("alpha", C.c_double), ("beta", C.c_double), ("gamma", C.c_double),
                ("max_log_scale", C.c_double), ("iterations", C.c_int),
                ("seed", C.c_uint64)]


class _Matrix(C.Structure):
    _fields_ = [("m", C.c_int64), ("n", C.c_int64), ("row_ptr", _i64p),
                ("col", _i32p), ("val", _dp), ("dense", _dp)]


class _Scaling(C.Structure):
    _fields_ = [("u", _dp), ("v", _dp), ("d", _dp), ("e", _dp),
                ("alpha", C.c_double), ("beta", C.c_double),
                ("box_feasible", C.c_int), ("iterate_bound_ok", C.c_int),
                ("apply_count", C.c_longlong), ("adjoint_count", C.c_longlong),
                ("hist_iter", _ip), ("hist_objective", _dp), ("hist_rms", _dp),
                ("hist_len", C.c_int), ("traj_u", _dp), ("traj_v", _dp)]


class _Lsqr(C.Structure):
    _fields_ = [("x", _dp), ("residual_history", _dp), ("hist_len", C.c_int),
                ("iterations", C.c_int), ("equil_iterations", C.c_int),
                ("reached_tol", C.c_int), ("breakdown", C.c_int),
                ("apply_count", C.c_longlong), ("adjoint_count", C.c_longlong),
                ("d", _dp), ("e", _dp)]


class _RefSgd(C.Structure):
    _fields_ = [("u", _dp), ("v", _dp), ("d", _dp), ("e", _dp),
                ("alpha", C.c_double), ("beta", C.c_double),
                ("box_feasible", C.c_int), ("iterate_bound_ok", C.c_int),
                ("apply_count", C.c_longlong), ("adjoint_count", C.c_longlong),
                ("hist_iter", _ip), ("hist_objective", _dp), ("hist_rms", _dp),
                ("hist_len", C.c_int)]


class _RefLsqr(C.Structure):
    _fields_ = [("x", _dp), ("residual_history", _dp), ("hist_len", C.c_int),
                ("iterations", C.c_int), ("equil_iterations", C.c_int),
                ("reached_tol", C.c_int), ("breakdown", C.c_int),
                ("apply_count", C.c_longlong), ("adjoint_count", C.c_longlong)]


@dataclass
class Scaling:
    u: np.ndarray
    v: np.ndarray
    d: np.ndarray
    e: np.ndarray
    alpha: float
    beta: float
    box_feasible: bool
    iterate_bound_ok: bool
    apply_count: int
    adjoint_count: int
    hist_iter: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    hist_objective: np.ndarray = field(default_factory=lambda: np.zeros(0))
    hist_rms: np.ndarray = field(default_factory=lambda: np.zeros(0))
    traj_u: np.ndarray | None = None
    traj_v: np.ndarray | None = None


@dataclass
class LsqrRun:
    x: np.ndarray
    residual_history: np.ndarray
    iterations: int
    equil_iterations: int
    reached_tol: bool
    breakdown: bool
    apply_count: int
    adjoint_count: int
    d: np.ndarray | None = None
    e: np.ndarray | None = None


class _CcpOpts(C.Structure):
    _fields_ = [("max_iters", C.c_int), ("tau", C.c_double), ("sigma", C.c_double),
                ("theta", C.c_double), ("p_star", C.c_double), ("gap_tol", C.c_double)]


class _CcpRun(C.Structure):  # eo_ccp_run and er_ccp_out share this layout
    _fields_ = [("x", _dp), ("obj_hist", _dp), ("gap_hist", _dp), ("hist_len", C.c_int),
                ("gap_len", C.c_int), ("tau", C.c_double), ("sigma", C.c_double),
                ("theta", C.c_double), ("iterations", C.c_int),
                ("equil_iterations", C.c_int), ("reached_tol", C.c_int),
                ("apply_count", C.c_longlong), ("adjoint_count", C.c_longlong)]


@dataclass
class CcpRun:
    x: np.ndarray
    objective_history: np.ndarray
    gap_history: np.ndarray
    tau: float
    sigma: float
    theta: float
    iterations: int
    equil_iterations: int
    reached_tol: bool
    apply_count: int
    adjoint_count: int


def _ccp_call(n, cap, fn):
    x, oh, gh = np.zeros(n), np.zeros(cap), np.zeros(cap)
    r = _CcpRun(ptr(x, _dp), ptr(oh, _dp), ptr(gh, _dp), 0, 0, 0.0, 0.0, 0.0, 0, 0, 0, 0, 0)
    rc = fn(C.byref(r))
    return rc, CcpRun(x, oh[:r.hist_len].copy(), gh[:r.gap_len].copy(), r.tau, r.sigma, r.theta,
                      r.iterations, r.equil_iterations, bool(r.reached_tol), r.apply_count,
                      r.adjoint_count)


class OracleError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class CsrArrays:
    """Host CSR (int64 row_ptr, int32 col, float64 val) or dense row-major."""

    def __init__(self, m, n, row_ptr=None, col=None, val=None, dense=None):
        self.m, self.n = int(m), int(n)
        self.row_ptr = None if row_ptr is None else np.ascontiguousarray(row_ptr, np.int64)
        self.col = None if col is None else np.ascontiguousarray(col, np.int32)
        self.val = None if val is None else np.ascontiguousarray(val, np.float64)
        self.dense = None if dense is None else np.ascontiguousarray(dense, np.float64)

    @property
    def nnz(self) -> int:
        return self.m * self.n if self.dense is not None else int(self.row_ptr[-1])

    def _struct(self):
        return _Matrix(self.m, self.n, ptr(self.row_ptr, _i64p), ptr(self.col, _i32p),
                       ptr(self.val, _dp), ptr(self.dense, _dp))


class _COracle:
    def __init__(self, path=LIB_PATH):
        if not os.path.exists(path):
            build(ref=False)
        L = C.CDLL(path)
        self.L = L
        L.eo_rng_next_u64.restype = C.c_uint64
        L.eo_mixed_seed.restype = C.c_uint64
        L.eo_mixed_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.eo_rng_init.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64]
        L.eo_mt64_seed.argtypes = [C.c_void_p, C.c_uint64]
        L.eo_rng_next_u64.argtypes = [C.c_void_p]
        L.eo_rng_uniform01.restype = C.c_double
        L.eo_rng_uniform01.argtypes = [C.c_void_p]
        L.eo_rng_normal.restype = C.c_double
        L.eo_rng_normal.argtypes = [C.c_void_p]
        L.eo_raw_outputs.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, _u64p]
        L.eo_sign_bits.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, _u32p]
        L.eo_rng_state.argtypes = [C.c_uint64, C.c_uint64, _u64p]
        L.eo_det_exp.restype = C.c_double
        L.eo_det_exp.argtypes = [C.c_double]
        for f in ("eo_canon_sum", "eo_canon_sumsq"):
            getattr(L, f).restype = C.c_double
            getattr(L, f).argtypes = [_dp, C.c_int64]
        L.eo_canon_dot.restype = C.c_double
        L.eo_canon_dot.argtypes = [_dp, _dp, C.c_int64]
        L.eo_csr_transpose.argtypes = [C.c_int64, C.c_int64, _i64p, _i32p, _dp, _i64p, _i32p, _dp]
        L.eo_csr_apply.argtypes = [C.c_int64, _i64p, _i32p, _dp, _dp, _dp]
        L.eo_csr_apply_adjoint.argtypes = [C.c_int64, C.c_int64, _i64p, _i32p, _dp, _dp, _dp]
        L.eo_dense_apply.argtypes = [C.c_int64, C.c_int64, _dp, _dp, _dp]
        L.eo_dense_apply_adjoint.argtypes = [C.c_int64, C.c_int64, _dp, _dp, _dp]
        L.eo_last_error.restype = C.c_char_p
        L.eo_sgd_equilibrate.argtypes = [C.POINTER(_Matrix), C.POINTER(_Params), C.c_int,
                                         C.POINTER(_Scaling)]
        L.eo_sgd_equilibrate_targets.argtypes = [C.POINTER(_Matrix), _dp, _dp, C.POINTER(_Params),
                                                 C.c_int, C.POINTER(_Scaling)]
        L.eo_sgd_equilibrate_symmetric.argtypes = [C.POINTER(_Matrix), C.POINTER(_Params),
                                                   C.c_int, C.POINTER(_Scaling)]
        L.eo_sgd_equilibrate_block.argtypes = [C.POINTER(_Matrix), _i64p, _i64p, C.c_int64,
                                               C.c_int64, C.POINTER(_Params), C.c_int,
                                               C.POINTER(_Scaling)]
        L.eo_spectral_norm.argtypes = [C.POINTER(_Matrix), C.c_int, C.c_double, C.c_uint64, _dp]
        L.eo_lasso_objective.restype = C.c_double
        L.eo_lasso_objective.argtypes = [C.POINTER(_Matrix), _dp, C.c_double, _dp]
        L.eo_ccp_lasso.argtypes = [C.POINTER(_Matrix), _dp, C.c_double, C.POINTER(_CcpOpts),
                                   C.POINTER(_CcpRun)]
        L.eo_ccp_lasso_preconditioned.argtypes = [C.POINTER(_Matrix), _dp, C.c_double,
                                                  C.POINTER(_Params), C.POINTER(_CcpOpts),
                                                  C.POINTER(_CcpRun)]
        L.eo_stochastic_gradient_estimate.argtypes = [C.POINTER(_Matrix), _dp, _dp,
                                                      C.POINTER(_Params), C.c_uint64, C.c_uint64,
                                                      C.c_uint64, _dp, _dp]
        L.eo_objective.restype = C.c_double
        L.eo_objective.argtypes = [C.POINTER(_Matrix), _dp, _dp, C.c_double, C.c_double, C.c_double]
        L.eo_rms_error.restype = C.c_double
        L.eo_rms_error.argtypes = [C.POINTER(_Matrix), _dp, _dp, C.c_double, C.c_double]
        L.eo_lsqr.argtypes = [C.POINTER(_Matrix), _dp, C.c_int, C.c_double, C.POINTER(_Lsqr)]
        L.eo_lsqr_preconditioned.argtypes = [C.POINTER(_Matrix), _dp, C.POINTER(_Params),
                                             C.c_int, C.c_double, C.POINTER(_Lsqr)]
        L.eo_resolve_targets.argtypes = [C.POINTER(_Params), C.c_int64, C.c_int64, _dp, _dp]

    # -- rng -------------------------------------------------------------
    def mixed_seed(self, seed, stream):
        return int(self.L.eo_mixed_seed(seed, stream))

    def raw_outputs(self, seed, stream, start, count):
        out = np.zeros(count, np.uint64)
        self.L.eo_raw_outputs(seed, stream, start, count, ptr(out, _u64p))
        return out

    def rng_state(self, seed, stream):
        out = np.zeros(312, np.uint64)
        self.L.eo_rng_state(seed, stream, ptr(out, _u64p))
        return out

    def sign_bits(self, seed, stream, start, count):
        out = np.zeros((count + 31) // 32, np.uint32)
        self.L.eo_sign_bits(seed, stream, start, count, ptr(out, _u32p))
        return out

    def mt64_std(self, seed, count):
        buf = C.create_string_buffer(312 * 8 + 64)
        self.L.eo_mt64_seed(buf, seed)
        return np.array([self.L.eo_rng_next_u64(buf) for _ in range(count)], np.uint64)

    def draws(self, seed, stream, kind, count):
        buf = C.create_string_buffer(312 * 8 + 64)
        self.L.eo_rng_init(buf, seed, stream)
        f = self.L.eo_rng_uniform01 if kind == "uniform" else self.L.eo_rng_normal
        return np.array([f(buf) for _ in range(count)])

    # -- numerics ---------------------------------------------------------
    def det_exp(self, x):
        x = np.ascontiguousarray(x, np.float64)
        return np.array([self.L.eo_det_exp(float(t)) for t in x.ravel()]).reshape(x.shape)

    def canon_sum(self, p):
        p = np.ascontiguousarray(p, np.float64)
        return self.L.eo_canon_sum(ptr(p, _dp), p.size)

    def canon_sumsq(self, p):
        p = np.ascontiguousarray(p, np.float64)
        return self.L.eo_canon_sumsq(ptr(p, _dp), p.size)

    def canon_dot(self, a, b):
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        return self.L.eo_canon_dot(ptr(a, _dp), ptr(b, _dp), a.size)

    # -- matrix -----------------------------------------------------------
    def transpose(self, A: CsrArrays) -> CsrArrays:
        trp = np.zeros(A.n + 1, np.int64)
        tc = np.zeros(A.nnz, np.int32)
        tv = np.zeros(A.nnz, np.float64)
        self.L.eo_csr_transpose(A.m, A.n, ptr(A.row_ptr, _i64p), ptr(A.col, _i32p),
                                ptr(A.val, _dp), ptr(trp, _i64p), ptr(tc, _i32p), ptr(tv, _dp))
        return CsrArrays(A.n, A.m, trp, tc, tv)

    def apply(self, A: CsrArrays, x, adjoint=False):
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros(A.n if adjoint else A.m)
        if A.dense is not None:
            f = self.L.eo_dense_apply_adjoint if adjoint else self.L.eo_dense_apply
            f(A.m, A.n, ptr(A.dense, _dp), ptr(x, _dp), ptr(y, _dp))
        elif adjoint:
            self.L.eo_csr_apply_adjoint(A.m, A.n, ptr(A.row_ptr, _i64p), ptr(A.col, _i32p),
                                        ptr(A.val, _dp), ptr(x, _dp), ptr(y, _dp))
        else:
            self.L.eo_csr_apply(A.m, ptr(A.row_ptr, _i64p), ptr(A.col, _i32p),
                                ptr(A.val, _dp), ptr(x, _dp), ptr(y, _dp))
        return y

    def _err(self, code):
        raise OracleError(code, self.L.eo_last_error().decode())

    def sgd_equilibrate(self, A: CsrArrays, alpha=0.0, beta=0.0, gamma=0.1,
                        max_log_scale=9.210340371976184, iterations=1000, seed=0,
                        diag_stride=0, trajectory=False) -> Scaling:
        m, n = A.m, A.n
        u, v, d, e = np.zeros(m), np.zeros(n), np.zeros(m), np.zeros(n)
        nh = iterations // diag_stride + 1 if diag_stride > 0 else 0
        hi, ho, hr = np.zeros(max(nh, 1), np.int32), np.zeros(max(nh, 1)), np.zeros(max(nh, 1))
        tu = np.zeros((iterations, m)) if trajectory else None
        tv = np.zeros((iterations, n)) if trajectory else None
        s = _Scaling(ptr(u, _dp), ptr(v, _dp), ptr(d, _dp), ptr(e, _dp), 0, 0, 0, 0, 0, 0,
                     ptr(hi, _ip), ptr(ho, _dp), ptr(hr, _dp), 0,
                     ptr(tu, _dp), ptr(tv, _dp))
        p = _Params(alpha, beta, gamma, max_log_scale, iterations, seed)
        mat = A._struct()
        rc = self.L.eo_sgd_equilibrate(C.byref(mat), C.byref(p), diag_stride, C.byref(s))
        if rc:
            self._err(rc)
        k = s.hist_len
        return Scaling(u, v, d, e, s.alpha, s.beta, bool(s.box_feasible),
                       bool(s.iterate_bound_ok), s.apply_count, s.adjoint_count,
                       hi[:k].copy(), ho[:k].copy(), hr[:k].copy(), tu, tv)

    def sgd_equilibrate_targets(self, A: CsrArrays, r, c, gamma=0.1,
                                max_log_scale=9.210340371976184, iterations=1000, seed=0,
                                diag_stride=0) -> Scaling:
        r = np.ascontiguousarray(r, np.float64)
        c = np.ascontiguousarray(c, np.float64)
        m, n = A.m, A.n
        u, v, d, e = np.zeros(m), np.zeros(n), np.zeros(m), np.zeros(n)
        nh = iterations // diag_stride + 1 if diag_stride > 0 else 1
        hi, ho, hr = np.zeros(nh, np.int32), np.zeros(nh), np.zeros(nh)
        s = _Scaling(ptr(u, _dp), ptr(v, _dp), ptr(d, _dp), ptr(e, _dp), 0, 0, 0, 0, 0, 0,
                     ptr(hi, _ip), ptr(ho, _dp), ptr(hr, _dp), 0, ptr(None, _dp),
                     ptr(None, _dp))
        p = _Params(0.0, 0.0, gamma, max_log_scale, iterations, seed)
        mat = A._struct()
        rc = self.L.eo_sgd_equilibrate_targets(C.byref(mat), ptr(r, _dp), ptr(c, _dp),
                                               C.byref(p), diag_stride, C.byref(s))
        if rc:
            self._err(rc)
        k = s.hist_len
        return Scaling(u, v, d, e, s.alpha, s.beta, bool(s.box_feasible),
                       bool(s.iterate_bound_ok), s.apply_count, s.adjoint_count,
                       hi[:k].copy(), ho[:k].copy(), hr[:k].copy())

    def _variant(self, call, m, n, iterations, diag_stride):
        u, v, d, e = np.zeros(m), np.zeros(n), np.zeros(m), np.zeros(n)
        nh = iterations // diag_stride + 1 if diag_stride > 0 else 1
        hi, ho, hr = np.zeros(nh, np.int32), np.zeros(nh), np.zeros(nh)
        s = _Scaling(ptr(u, _dp), ptr(v, _dp), ptr(d, _dp), ptr(e, _dp), 0, 0, 0, 0, 0, 0,
                     ptr(hi, _ip), ptr(ho, _dp), ptr(hr, _dp), 0, ptr(None, _dp),
                     ptr(None, _dp))
        rc = call(C.byref(s))
        if rc:
            self._err(rc)
        k = s.hist_len
        return Scaling(u, v, d, e, s.alpha, s.beta, bool(s.box_feasible),
                       bool(s.iterate_bound_ok), s.apply_count, s.adjoint_count,
                       hi[:k].copy(), ho[:k].copy(), hr[:k].copy())

    def sgd_equilibrate_symmetric(self, A: CsrArrays, alpha=0.0, beta=0.0, gamma=0.1,
                                  max_log_scale=9.210340371976184, iterations=1000, seed=0,
                                  diag_stride=0) -> Scaling:
        """src/variants.cpp:35-103"""
        p = _Params(alpha, beta, gamma, max_log_scale, iterations, seed)
        mat = A._struct()
        return self._variant(lambda s: self.L.eo_sgd_equilibrate_symmetric(
            C.byref(mat), C.byref(p), diag_stride, s), A.m, A.n, iterations, diag_stride)

    def sgd_equilibrate_block(self, A: CsrArrays, row_block, col_block, row_blocks, col_blocks,
                              gamma=0.1, max_log_scale=9.210340371976184, iterations=1000,
                              seed=0, diag_stride=0) -> Scaling:
        """src/variants.cpp:156-240"""
        rb = np.ascontiguousarray(row_block, np.int64)
        cb = np.ascontiguousarray(col_block, np.int64)
        p = _Params(0.0, 0.0, gamma, max_log_scale, iterations, seed)
        mat = A._struct()
        return self._variant(lambda s: self.L.eo_sgd_equilibrate_block(
            C.byref(mat), ptr(rb, _i64p), ptr(cb, _i64p), row_blocks, col_blocks, C.byref(p),
            diag_stride, s), A.m, A.n, iterations, diag_stride)

    def stochastic_gradient_estimate(self, A: CsrArrays, u, v, seed, stream, offset, alpha=0.0,
                                     beta=0.0, gamma=0.1):
        """src/equilibrate.cpp:60-71"""
        u = np.ascontiguousarray(u, np.float64)
        v = np.ascontiguousarray(v, np.float64)
        gu, gv = np.zeros(A.m), np.zeros(A.n)
        p = _Params(alpha, beta, gamma, 9.210340371976184, 1, 0)
        mat = A._struct()
        rc = self.L.eo_stochastic_gradient_estimate(C.byref(mat), ptr(u, _dp), ptr(v, _dp),
                                                    C.byref(p), seed, stream, offset,
                                                    ptr(gu, _dp), ptr(gv, _dp))
        if rc:
            self._err(rc)
        return gu, gv

    def spectral_norm(self, A: CsrArrays, max_iters=100, rel_tol=1e-9, seed=0) -> float:
        """src/lsqr.cpp:140-163"""
        out = C.c_double(0.0)
        mat = A._struct()
        rc = self.L.eo_spectral_norm(C.byref(mat), max_iters, rel_tol, seed, C.byref(out))
        if rc:
            self._err(rc)
        return out.value

    def lasso_objective(self, A: CsrArrays, b, lam, x) -> float:
        mat = A._struct()
        return self.L.eo_lasso_objective(C.byref(mat), ptr(np.ascontiguousarray(b, np.float64),
                                                            _dp), lam,
                                         ptr(np.ascontiguousarray(x, np.float64), _dp))

    def ccp_lasso(self, A: CsrArrays, b, lam, max_iters=1000, tau=0.0, sigma=0.0, theta=1.0,
                  p_star=float("nan"), gap_tol=0.0, params=None) -> CcpRun:
        """ccp_lasso / ccp_lasso_preconditioned (src/ccp.cpp:125-141);
        params = dict of EquilibrationParams fields selects the latter."""
        b = np.ascontiguousarray(b, np.float64)
        o = _CcpOpts(max_iters, tau, sigma, theta, p_star, gap_tol)
        mat = A._struct()
        T = params.get("iterations", 1000) if params is not None else 0
        cap = max(max_iters, 0) + 1 + max(T, 0)
        if params is None:
            rc, run = _ccp_call(A.n, cap, lambda r: self.L.eo_ccp_lasso(
                C.byref(mat), ptr(b, _dp), lam, C.byref(o), r))
        else:
            p = _Params(params.get("alpha", 0.0), params.get("beta", 0.0),
                        params.get("gamma", 0.1), params.get("max_log_scale", 9.210340371976184),
                        T, params.get("seed", 0))
            rc, run = _ccp_call(A.n, cap, lambda r: self.L.eo_ccp_lasso_preconditioned(
                C.byref(mat), ptr(b, _dp), lam, C.byref(p), C.byref(o), r))
        if rc:
            self._err(rc)
        return run

    def objective(self, A, u, v, alpha2, beta2, gamma):
        mat = A._struct()
        return self.L.eo_objective(C.byref(mat), ptr(np.ascontiguousarray(u, np.float64), _dp),
                                   ptr(np.ascontiguousarray(v, np.float64), _dp),
                                   alpha2, beta2, gamma)

    def rms_error(self, A, u, v, alpha, beta):
        mat = A._struct()
        return self.L.eo_rms_error(C.byref(mat), ptr(np.ascontiguousarray(u, np.float64), _dp),
                                   ptr(np.ascontiguousarray(v, np.float64), _dp), alpha, beta)

    def _lsqr_struct(self, A, cap, want_de):
        x = np.zeros(A.n)
        h = np.zeros(cap)
        d = np.zeros(A.m) if want_de else None
        e = np.zeros(A.n) if want_de else None
        return x, h, d, e, _Lsqr(ptr(x, _dp), ptr(h, _dp), 0, 0, 0, 0, 0, 0, 0,
                                 ptr(d, _dp), ptr(e, _dp))

    def lsqr(self, A, b, max_iters, tol) -> LsqrRun:
        b = np.ascontiguousarray(b, np.float64)
        x, h, _, _, r = self._lsqr_struct(A, max_iters + 1, False)
        mat = A._struct()
        rc = self.L.eo_lsqr(C.byref(mat), ptr(b, _dp), max_iters, tol, C.byref(r))
        if rc:
            self._err(rc)
        return LsqrRun(x, h[:r.hist_len].copy(), r.iterations, r.equil_iterations,
                       bool(r.reached_tol), bool(r.breakdown), r.apply_count, r.adjoint_count)

    def lsqr_preconditioned(self, A, b, max_iters, tol, alpha=0.0, beta=0.0, gamma=0.1,
                            max_log_scale=9.210340371976184, iterations=1000,
                            seed=0) -> LsqrRun:
        b = np.ascontiguousarray(b, np.float64)
        x, h, d, e, r = self._lsqr_struct(A, max_iters + iterations + 2, True)
        p = _Params(alpha, beta, gamma, max_log_scale, iterations, seed)
        mat = A._struct()
        rc = self.L.eo_lsqr_preconditioned(C.byref(mat), ptr(b, _dp), C.byref(p), max_iters,
                                           tol, C.byref(r))
        if rc:
            self._err(rc)
        return LsqrRun(x, h[:r.hist_len].copy(), r.iterations, r.equil_iterations,
                       bool(r.reached_tol), bool(r.breakdown), r.apply_count,
                       r.adjoint_count, d, e)


class _RefOracle:
    """The reference's own sources (oracle/_ref/libequil_ref.so)."""

    def __init__(self, path=REF_PATH):
        if not os.path.exists(path):
            build(ref=True)
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = C.CDLL(path)
        self.L = L
        L.er_last_error.restype = C.c_char_p
        L.er_rng_outputs.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, _u64p]
        L.er_rng_draws.argtypes = [C.c_uint64, C.c_uint64, C.c_int, C.c_uint64, _dp]
        L.er_matrix_csr.argtypes = [C.c_int64, C.c_int64, _i64p, _i32p, _dp, C.POINTER(C.c_void_p)]
        L.er_matrix_coo.argtypes = [C.c_int64, C.c_int64, C.c_int64, _i64p, _i64p, _dp,
                                    C.POINTER(C.c_void_p)]
        L.er_matrix_dense.argtypes = [C.c_int64, C.c_int64, _dp, C.POINTER(C.c_void_p)]
        L.er_matrix_free.argtypes = [C.c_void_p]
        L.er_mm_read.argtypes = [C.c_char_p, C.POINTER(C.c_void_p), _i64p, _i64p,
                                 C.POINTER(C.c_int)]
        L.er_mm_write.argtypes = [C.c_void_p, C.c_char_p]
        L.er_matrix_to_dense.argtypes = [C.c_void_p, _dp]
        L.er_matrix_nnz.argtypes = [C.c_void_p]
        L.er_matrix_nnz.restype = C.c_int64
        L.er_matrix_export.argtypes = [C.c_void_p, _i64p, _i32p, _dp]
        L.er_matrix_transposed.argtypes = [C.c_void_p]
        L.er_matrix_transposed.restype = C.c_void_p
        L.er_apply.argtypes = [C.c_void_p, _dp, _dp, C.c_int]
        L.er_sgd_equilibrate.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_double,
                                         C.c_double, C.c_int, C.c_uint64, C.c_int,
                                         C.POINTER(_RefSgd)]
        L.er_sgd_targets.argtypes = [C.c_void_p, _dp, _dp, C.c_double, C.c_double, C.c_int,
                                     C.c_uint64, C.c_int, C.POINTER(_RefSgd)]
        L.er_sgd_symmetric.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_double,
                                       C.c_double, C.c_int, C.c_uint64, C.c_int,
                                       C.POINTER(_RefSgd)]
        L.er_sgd_block.argtypes = [C.c_void_p, _i64p, _i64p, C.c_int64, C.c_int64, C.c_double,
                                   C.c_double, C.c_int, C.c_uint64, C.c_int, C.POINTER(_RefSgd)]
        L.er_ccp_lasso.argtypes = [C.c_void_p, _dp, C.c_double, C.c_int, C.c_double,
                                   C.c_double, C.c_double, C.c_double, C.c_double,
                                   C.POINTER(_CcpRun)]
        L.er_ccp_lasso_preconditioned.argtypes = [
            C.c_void_p, _dp, C.c_double, C.c_double, C.c_double, C.c_double, C.c_double,
            C.c_int, C.c_uint64, C.c_int, C.c_double, C.c_double, C.c_double, C.c_double,
            C.c_double, C.POINTER(_CcpRun)]
        L.er_spectral_norm.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_uint64, _dp]
        L.er_lasso_objective.argtypes = [C.c_void_p, _dp, C.c_double, _dp, _dp]
        L.er_lasso_fista.argtypes = [C.c_void_p, _dp, C.c_double, C.c_double, C.c_int, _dp, _dp]
        L.er_objective.argtypes = [C.c_void_p, _dp, _dp, C.c_double, C.c_double, C.c_double, _dp]
        L.er_gradient.argtypes = [C.c_void_p, _dp, _dp, C.c_double, C.c_double, C.c_double, _dp,
                                  _dp]
        L.er_sge.argtypes = [C.c_void_p, _dp, _dp, C.c_double, C.c_double, C.c_double,
                             C.c_uint64, C.c_uint64, C.c_uint64, _dp, _dp]
        L.er_lsqr.argtypes = [C.c_void_p, _dp, C.c_int, C.c_double, C.POINTER(_RefLsqr)]
        L.er_lsqr_preconditioned.argtypes = [C.c_void_p, _dp, C.c_double, C.c_double,
                                             C.c_double, C.c_double, C.c_int, C.c_uint64,
                                             C.c_int, C.c_double, C.POINTER(_RefLsqr)]
        L.er_rms_error.restype = C.c_double
        L.er_rms_error.argtypes = [C.c_void_p, _dp, _dp, C.c_double, C.c_double]

    def _err(self, code):
        raise OracleError(code, self.L.er_last_error().decode())

    def outputs(self, seed, stream, count):
        out = np.zeros(count, np.uint64)
        self.L.er_rng_outputs(seed, stream, count, ptr(out, _u64p))
        return out

    def draws(self, seed, stream, kind, count):
        out = np.zeros(count)
        self.L.er_rng_draws(seed, stream, {"uniform": 0, "normal": 1, "sign": 2}[kind],
                            count, ptr(out, _dp))
        return out

    def matrix(self, A: CsrArrays):
        h = C.c_void_p()
        if A.dense is not None:
            rc = self.L.er_matrix_dense(A.m, A.n, ptr(A.dense, _dp), C.byref(h))
        else:
            rc = self.L.er_matrix_csr(A.m, A.n, ptr(A.row_ptr, _i64p), ptr(A.col, _i32p),
                                      ptr(A.val, _dp), C.byref(h))
        if rc:
            self._err(rc)
        return RefMatrix(self, h, A.m, A.n)

    def read_matrix_market(self, path):
        """(RefMatrix, is_sparse) from the reference's read_matrix_market_file."""
        h, m, n, sp = C.c_void_p(), C.c_int64(), C.c_int64(), C.c_int()
        rc = self.L.er_mm_read(str(path).encode(), C.byref(h), C.byref(m), C.byref(n),
                               C.byref(sp))
        if rc:
            self._err(rc)
        return RefMatrix(self, h, m.value, n.value), bool(sp.value)

    def matrix_coo(self, m, n, rows, cols, vals):
        rows = np.ascontiguousarray(rows, np.int64)
        cols = np.ascontiguousarray(cols, np.int64)
        vals = np.ascontiguousarray(vals, np.float64)
        h = C.c_void_p()
        rc = self.L.er_matrix_coo(m, n, rows.size, ptr(rows, _i64p), ptr(cols, _i64p),
                                  ptr(vals, _dp), C.byref(h))
        if rc:
            self._err(rc)
        return RefMatrix(self, h, m, n)


class RefMatrix:
    def __init__(self, R: _RefOracle, h, m, n):
        self.R, self.h, self.m, self.n = R, h, m, n

    def write_matrix_market(self, path):
        rc = self.R.L.er_mm_write(self.h, str(path).encode())
        if rc:
            self.R._err(rc)

    def to_dense(self):
        out = np.zeros((self.m, self.n))
        rc = self.R.L.er_matrix_to_dense(self.h, ptr(out, _dp))
        if rc:
            self.R._err(rc)
        return out

    def __del__(self):
        try:
            self.R.L.er_matrix_free(self.h)
        except Exception:
            pass

    def export(self) -> CsrArrays:
        nnz = self.R.L.er_matrix_nnz(self.h)
        rp = np.zeros(self.m + 1, np.int64)
        c = np.zeros(nnz, np.int32)
        v = np.zeros(nnz)
        self.R.L.er_matrix_export(self.h, ptr(rp, _i64p), ptr(c, _i32p), ptr(v, _dp))
        return CsrArrays(self.m, self.n, rp, c, v)

    def transposed(self) -> "RefMatrix":
        return RefMatrix(self.R, C.c_void_p(self.R.L.er_matrix_transposed(self.h)),
                         self.n, self.m)

    def apply(self, x, adjoint=False):
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros(self.n if adjoint else self.m)
        rc = self.R.L.er_apply(self.h, ptr(x, _dp), ptr(y, _dp), int(adjoint))
        if rc:
            self.R._err(rc)
        return y

    def sgd_equilibrate(self, alpha=0.0, beta=0.0, gamma=0.1,
                        max_log_scale=9.210340371976184, iterations=1000, seed=0,
                        diag_stride=0) -> Scaling:
        u, v, d, e = np.zeros(self.m), np.zeros(self.n), np.zeros(self.m), np.zeros(self.n)
        nh = iterations // diag_stride + 1 if diag_stride > 0 else 1
        hi, ho, hr = np.zeros(nh, np.int32), np.zeros(nh), np.zeros(nh)
        s = _RefSgd(ptr(u, _dp), ptr(v, _dp), ptr(d, _dp), ptr(e, _dp), 0, 0, 0, 0, 0, 0,
                    ptr(hi, _ip), ptr(ho, _dp), ptr(hr, _dp), 0)
        rc = self.R.L.er_sgd_equilibrate(self.h, alpha, beta, gamma, max_log_scale,
                                         iterations, seed, diag_stride, C.byref(s))
        if rc:
            self.R._err(rc)
        k = s.hist_len
        return Scaling(u, v, d, e, s.alpha, s.beta, bool(s.box_feasible),
                       bool(s.iterate_bound_ok), s.apply_count, s.adjoint_count,
                       hi[:k].copy(), ho[:k].copy(), hr[:k].copy())

    def sgd_equilibrate_targets(self, r, c, gamma=0.1, max_log_scale=9.210340371976184,
                                iterations=1000, seed=0, diag_stride=0) -> Scaling:
        r = np.ascontiguousarray(r, np.float64)
        c = np.ascontiguousarray(c, np.float64)
        u, v, d, e = np.zeros(self.m), np.zeros(self.n), np.zeros(self.m), np.zeros(self.n)
        nh = iterations // diag_stride + 1 if diag_stride > 0 else 1
        hi, ho, hr = np.zeros(nh, np.int32), np.zeros(nh), np.zeros(nh)
        s = _RefSgd(ptr(u, _dp), ptr(v, _dp), ptr(d, _dp), ptr(e, _dp), 0, 0, 0, 0, 0, 0,
                    ptr(hi, _ip), ptr(ho, _dp), ptr(hr, _dp), 0)
        rc = self.R.L.er_sgd_targets(self.h, ptr(r, _dp), ptr(c, _dp), gamma, max_log_scale,
                                     iterations, seed, diag_stride, C.byref(s))
        if rc:
            self.R._err(rc)
        k = s.hist_len
        return Scaling(u, v, d, e, s.alpha, s.beta, bool(s.box_feasible),
                       bool(s.iterate_bound_ok), s.apply_count, s.adjoint_count,
                       hi[:k].copy(), ho[:k].copy(), hr[:k].copy())

    def _variant(self, call, iterations, diag_stride):
        u, v, d, e = np.zeros(self.m), np.zeros(self.n), np.zeros(self.m), np.zeros(self.n)
        nh = iterations // diag_stride + 1 if diag_stride > 0 else 1
        hi, ho, hr = np.zeros(nh, np.int32), np.zeros(nh), np.zeros(nh)
        s = _RefSgd(ptr(u, _dp), ptr(v, _dp), ptr(d, _dp), ptr(e, _dp), 0, 0, 0, 0, 0, 0,
                    ptr(hi, _ip), ptr(ho, _dp), ptr(hr, _dp), 0)
        rc = call(C.byref(s))
        if rc:
            self.R._err(rc)
        k = s.hist_len
        return Scaling(u, v, d, e, s.alpha, s.beta, bool(s.box_feasible),
                       bool(s.iterate_bound_ok), s.apply_count, s.adjoint_count,
                       hi[:k].copy(), ho[:k].copy(), hr[:k].copy())

    def sgd_equilibrate_symmetric(self, alpha=0.0, beta=0.0, gamma=0.1,
                                  max_log_scale=9.210340371976184, iterations=1000, seed=0,
                                  diag_stride=0) -> Scaling:
        return self._variant(lambda s: self.R.L.er_sgd_symmetric(
            self.h, alpha, beta, gamma, max_log_scale, iterations, seed, diag_stride, s),
            iterations, diag_stride)

    def sgd_equilibrate_block(self, row_block, col_block, row_blocks, col_blocks, gamma=0.1,
                              max_log_scale=9.210340371976184, iterations=1000, seed=0,
                              diag_stride=0) -> Scaling:
        rb = np.ascontiguousarray(row_block, np.int64)
        cb = np.ascontiguousarray(col_block, np.int64)
        return self._variant(lambda s: self.R.L.er_sgd_block(
            self.h, ptr(rb, _i64p), ptr(cb, _i64p), row_blocks, col_blocks, gamma,
            max_log_scale, iterations, seed, diag_stride, s), iterations, diag_stride)

    def ccp_lasso(self, b, lam, max_iters=1000, tau=0.0, sigma=0.0, theta=1.0,
                  p_star=float("nan"), gap_tol=0.0, params=None) -> CcpRun:
        b = np.ascontiguousarray(b, np.float64)
        T = params.get("iterations", 1000) if params is not None else 0
        cap = max(max_iters, 0) + 1 + max(T, 0)
        if params is None:
            rc, run = _ccp_call(self.n, cap, lambda r: self.R.L.er_ccp_lasso(
                self.h, ptr(b, _dp), lam, max_iters, tau, sigma, theta, p_star, gap_tol, r))
        else:
            rc, run = _ccp_call(self.n, cap, lambda r: self.R.L.er_ccp_lasso_preconditioned(
                self.h, ptr(b, _dp), lam, params.get("alpha", 0.0), params.get("beta", 0.0),
                params.get("gamma", 0.1), params.get("max_log_scale", 9.210340371976184), T,
                params.get("seed", 0), max_iters, tau, sigma, theta, p_star, gap_tol, r))
        if rc:
            self.R._err(rc)
        return run

    def objective(self, u, v, alpha=0.0, beta=0.0, gamma=0.1) -> float:
        out = C.c_double(0.0)
        rc = self.R.L.er_objective(self.h, ptr(np.ascontiguousarray(u, np.float64), _dp),
                                   ptr(np.ascontiguousarray(v, np.float64), _dp), alpha, beta,
                                   gamma, C.byref(out))
        if rc:
            self.R._err(rc)
        return out.value

    def gradient(self, u, v, alpha=0.0, beta=0.0, gamma=0.1):
        gu, gv = np.zeros(self.m), np.zeros(self.n)
        rc = self.R.L.er_gradient(self.h, ptr(np.ascontiguousarray(u, np.float64), _dp),
                                  ptr(np.ascontiguousarray(v, np.float64), _dp), alpha, beta,
                                  gamma, ptr(gu, _dp), ptr(gv, _dp))
        if rc:
            self.R._err(rc)
        return gu, gv

    def stochastic_gradient_estimate(self, u, v, seed, stream, offset, alpha=0.0, beta=0.0,
                                     gamma=0.1):
        gu, gv = np.zeros(self.m), np.zeros(self.n)
        rc = self.R.L.er_sge(self.h, ptr(np.ascontiguousarray(u, np.float64), _dp),
                             ptr(np.ascontiguousarray(v, np.float64), _dp), alpha, beta, gamma,
                             seed, stream, offset, ptr(gu, _dp), ptr(gv, _dp))
        if rc:
            self.R._err(rc)
        return gu, gv

    def spectral_norm(self, max_iters=100, rel_tol=1e-9, seed=0) -> float:
        out = C.c_double(0.0)
        rc = self.R.L.er_spectral_norm(self.h, max_iters, rel_tol, seed, C.byref(out))
        if rc:
            self.R._err(rc)
        return out.value

    def lasso_objective(self, b, lam, x) -> float:
        out = C.c_double(0.0)
        rc = self.R.L.er_lasso_objective(self.h, ptr(np.ascontiguousarray(b, np.float64), _dp),
                                         lam, ptr(np.ascontiguousarray(x, np.float64), _dp),
                                         C.byref(out))
        if rc:
            self.R._err(rc)
        return out.value

    def lasso_fista(self, b, lam, grad_map_tol=1e-12, max_iters=500000):
        x, ps = np.zeros(self.n), C.c_double(0.0)
        rc = self.R.L.er_lasso_fista(self.h, ptr(np.ascontiguousarray(b, np.float64), _dp), lam,
                                     grad_map_tol, max_iters, ptr(x, _dp), C.byref(ps))
        if rc:
            self.R._err(rc)
        return x, ps.value

    def lsqr(self, b, max_iters, tol) -> LsqrRun:
        b = np.ascontiguousarray(b, np.float64)
        x, h = np.zeros(self.n), np.zeros(max_iters + 1)
        r = _RefLsqr(ptr(x, _dp), ptr(h, _dp), 0, 0, 0, 0, 0, 0, 0)
        rc = self.R.L.er_lsqr(self.h, ptr(b, _dp), max_iters, tol, C.byref(r))
        if rc:
            self.R._err(rc)
        return LsqrRun(x, h[:r.hist_len].copy(), r.iterations, r.equil_iterations,
                       bool(r.reached_tol), bool(r.breakdown), r.apply_count, r.adjoint_count)

    def lsqr_preconditioned(self, b, max_iters, tol, alpha=0.0, beta=0.0, gamma=0.1,
                            max_log_scale=9.210340371976184, iterations=1000,
                            seed=0) -> LsqrRun:
        b = np.ascontiguousarray(b, np.float64)
        x, h = np.zeros(self.n), np.zeros(max_iters + iterations + 2)
        r = _RefLsqr(ptr(x, _dp), ptr(h, _dp), 0, 0, 0, 0, 0, 0, 0)
        rc = self.R.L.er_lsqr_preconditioned(self.h, ptr(b, _dp), alpha, beta, gamma,
                                             max_log_scale, iterations, seed, max_iters, tol,
                                             C.byref(r))
        if rc:
            self.R._err(rc)
        return LsqrRun(x, h[:r.hist_len].copy(), r.iterations, r.equil_iterations,
                       bool(r.reached_tol), bool(r.breakdown), r.apply_count, r.adjoint_count)

    def rms_error(self, u, v, alpha, beta):
        return self.R.L.er_rms_error(self.h, ptr(np.ascontiguousarray(u, np.float64), _dp),
                                     ptr(np.ascontiguousarray(v, np.float64), _dp), alpha, beta)


_C = None
_R = None


def c_oracle() -> _COracle:
    global _C
    if _C is None:
        _C = _COracle()
    return _C


def ref_oracle() -> _RefOracle:
    global _R
    if _R is None:
        _R = _RefOracle()
    return _R


def ref_available() -> bool:
    return os.path.exists(REF_PATH) or os.path.isdir(REFERENCE_SRC)
