"""Python mirror of the reference's interface for the equilibration hot path.

Same names, argument meaning and error behaviour as the reference's C++ API
(include/equil/{params,explicit_matrix,equilibrate,lsqr}.hpp); every call goes
through the C ABI of libequil_b200.so (include/equil_b200.h) and runs on the
GPU.  ``InvalidArgument`` stands for std::invalid_argument (detail::require),
``EquilRuntimeError`` for std::runtime_error (detail::check).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib as L

K_AUTO_TARGET = 0.0
DEFAULT_MAX_LOG_SCALE = 9.210340371976184  # log(1e4), include/equil/params.hpp:20
SGD_PROBE_STREAM = 17                      # include/equil/streams.hpp:17


class InvalidArgument(ValueError):
    """std::invalid_argument (include/equil/common.hpp:16-18)."""


class EquilRuntimeError(RuntimeError):
    """std::runtime_error (include/equil/common.hpp:20-22) and CUDA/NCCL failures."""


def _check(rc: int) -> None:
    if rc == L.EQUIL_OK:
        return
    msg = L.load().equil_last_error().decode()
    if rc == L.EQUIL_EINVAL:
        raise InvalidArgument(msg)
    raise EquilRuntimeError(f"[status {rc}] {msg}")


@dataclass
class EquilibrationParams:
    """include/equil/params.hpp:14-23."""
    alpha: float = K_AUTO_TARGET
    beta: float = K_AUTO_TARGET
    gamma: float = 0.1
    max_log_scale: float = DEFAULT_MAX_LOG_SCALE
    iterations: int = 1000
    seed: int = 0

    def _c(self) -> L.Params:
        return L.Params(self.alpha, self.beta, self.gamma, self.max_log_scale,
                        int(self.iterations), int(self.seed))


@dataclass
class DiagnosticsConfig:
    """include/equil/equilibrate.hpp:63-67 (``matrix`` is implicit: the
    operator being equilibrated; condition numbers are out of scope)."""
    stride: int = 1
    want_objective: bool = True
    want_rms: bool = True


@dataclass
class IterationRecord:
    """include/equil/equilibrate.hpp:51-56."""
    iter: int
    objective: Optional[float] = None
    rms: Optional[float] = None
    cond: Optional[float] = None


@dataclass
class ScalingResult:
    """include/equil/equilibrate.hpp:69-78."""
    u: np.ndarray
    v: np.ndarray
    d: np.ndarray
    e: np.ndarray
    alpha: float = 0.0
    beta: float = 0.0
    history: list = field(default_factory=list)
    box_feasible: bool = True
    iterate_bound_ok: bool = True
    apply_count: int = 0
    adjoint_count: int = 0


@dataclass
class LsqrRun:
    """include/equil/lsqr.hpp:10-23."""
    x: np.ndarray
    residual_history: list
    iterations: int = 0
    equil_iterations: int = 0
    reached_tol: bool = False
    breakdown: bool = False
    apply_count: int = 0
    adjoint_count: int = 0


def resolve_targets(params: EquilibrationParams, rows: int, cols: int):
    """src/params.cpp:7-33 -> (alpha, beta)."""
    a, b = C.c_double(), C.c_double()
    p = params._c()
    _check(L.load().equil_resolve_targets(C.byref(p), rows, cols, C.byref(a), C.byref(b)))
    return a.value, b.value


def validate_params(params: EquilibrationParams) -> None:
    """src/params.cpp:35-44."""
    p = params._c()
    _check(L.load().equil_validate_params(C.byref(p)))


class ExplicitMatrix:
    """Device-resident matrix behind the reference's ExplicitMatrix interface
    (include/equil/explicit_matrix.hpp:13-86): CSR(A) and CSR(A^T) (built on
    the device), or dense row-major.  Also the LinearOperator plugin
    (rows/cols/apply/apply_adjoint, include/equil/linop.hpp:13-25)."""

    def __init__(self, handle, m, n, nnz, dense):
        self._h = handle
        self._m, self._n, self._nnz, self._dense = m, n, nnz, dense

    # -- construction ------------------------------------------------------
    @staticmethod
    def from_csr(rows: int, cols: int, row_ptr, col, val, device: int = 0,
                 rank: int = 0, world_size: int = 1, nccl_id: bytes | None = None):
        """Canonical CSR (columns strictly ascending per row); validated and
        transposed on the device."""
        rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        c_in = np.asarray(col)
        if c_in.dtype != np.int32 and c_in.size:
            # wider indices must not wrap into range on the int32 cast: report
            # the first out-of-range entry as ExplicitMatrix::sparse does
            # (src/explicit_matrix.cpp:23-28)
            bad = np.flatnonzero((c_in < 0) | (c_in >= cols))
            if bad.size:
                k = int(bad[0])
                i = int(np.searchsorted(rp, k, side="right")) - 1
                raise InvalidArgument(f"ExplicitMatrix::sparse: entry ({i}, {int(c_in[k])}) "
                                      "out of range")
        ci = np.ascontiguousarray(c_in, dtype=np.int32)
        va = np.ascontiguousarray(val, dtype=np.float64)
        if rp.size != rows + 1 and rows > 0:
            raise InvalidArgument("ExplicitMatrix::sparse: row_ptr must have rows + 1 entries")
        idbuf = C.create_string_buffer(nccl_id, 128) if nccl_id else None
        cfg = L.DeviceCfg(device, rank, world_size,
                          C.cast(idbuf, C.c_void_p) if idbuf is not None else None)
        h = C.c_void_p()
        _check(L.load().equil_matrix_create_csr(rows, cols, L.ptr(rp, L._i64p),
                                                L.ptr(ci, L._i32p), L.ptr(va, L._dp),
                                                C.byref(cfg), C.byref(h)))
        return ExplicitMatrix(h, rows, cols, int(rp[-1]) if rows > 0 else 0, False)

    @staticmethod
    def sparse(rows: int, cols: int, entries, device: int = 0):
        """ExplicitMatrix::sparse (src/explicit_matrix.cpp:19-57): entries are
        (row, col, value) triples in any order (or a (rows, cols, vals) tuple of
        arrays).  On the device: range check in input order, sort by (row, col),
        duplicate rejection in sorted order, CSR, then CSR(A^T)."""
        if isinstance(entries, tuple) and len(entries) == 3 and hasattr(entries[0], "__len__"):
            r = np.ascontiguousarray(entries[0], dtype=np.int64)
            c = np.ascontiguousarray(entries[1], dtype=np.int64)
            v = np.ascontiguousarray(entries[2], dtype=np.float64)
        else:
            ent = list(entries)
            r = np.array([e[0] for e in ent], dtype=np.int64)
            c = np.array([e[1] for e in ent], dtype=np.int64)
            v = np.array([e[2] for e in ent], dtype=np.float64)
        cfg = L.DeviceCfg(device, 0, 1, None)
        h = C.c_void_p()
        _check(L.load().equil_matrix_create_coo(rows, cols, r.size, L.ptr(r, L._i64p),
                                                L.ptr(c, L._i64p), L.ptr(v, L._dp),
                                                C.byref(cfg), C.byref(h)))
        return ExplicitMatrix(h, rows, cols, int(r.size), False)

    @staticmethod
    def dense(values, device: int = 0):
        """ExplicitMatrix::dense (src/explicit_matrix.cpp:8-17)."""
        a = np.ascontiguousarray(values, dtype=np.float64)
        if a.ndim != 2 or a.shape[0] <= 0 or a.shape[1] <= 0:
            raise InvalidArgument("ExplicitMatrix::dense: dimensions must be positive")
        cfg = L.DeviceCfg(device, 0, 1, None)
        h = C.c_void_p()
        _check(L.load().equil_matrix_create_dense(a.shape[0], a.shape[1], L.ptr(a, L._dp),
                                                  C.byref(cfg), C.byref(h)))
        return ExplicitMatrix(h, a.shape[0], a.shape[1], a.size, True)

    @staticmethod
    def identity(n: int, device: int = 0):
        """ExplicitMatrix::identity (src/explicit_matrix.cpp:59-65)."""
        if n <= 0:
            raise InvalidArgument("ExplicitMatrix::identity: n must be positive")
        return ExplicitMatrix.from_csr(n, n, np.arange(n + 1), np.arange(n), np.ones(n), device)

    @staticmethod
    def _from_handle(h):
        m, n, nnz = C.c_int64(), C.c_int64(), C.c_int64()
        _check(L.load().equil_matrix_shape(h, C.byref(m), C.byref(n), C.byref(nnz)))
        return ExplicitMatrix(h, m.value, n.value, nnz.value,
                              bool(L.load().equil_matrix_is_dense(h)))

    @staticmethod
    def read_matrix_market(path: str, device: int = 0):
        """read_matrix_market_file (include/equil/matrix_market.hpp:17-18):
        parsed on host threads, sorted / validated / converted on the device."""
        cfg = L.DeviceCfg(device, 0, 1, None)
        h = C.c_void_p()
        _check(L.load().equil_matrix_read_matrix_market(str(path).encode(), C.byref(cfg),
                                                        C.byref(h)))
        return ExplicitMatrix._from_handle(h)

    def write_matrix_market(self, path: str):
        """write_matrix_market_file (include/equil/matrix_market.hpp:20-21)."""
        _check(L.load().equil_matrix_write_matrix_market(self._h, str(path).encode()))

    @staticmethod
    def load_binary(path: str, device: int = 0):
        """Binary CSR / dense file written by save_binary (fast reload)."""
        cfg = L.DeviceCfg(device, 0, 1, None)
        h = C.c_void_p()
        _check(L.load().equil_matrix_load_binary(str(path).encode(), C.byref(cfg), C.byref(h)))
        return ExplicitMatrix._from_handle(h)

    def save_binary(self, path: str):
        _check(L.load().equil_matrix_save_binary(self._h, str(path).encode()))

    def is_sparse(self) -> bool:
        return not self._dense

    def to_csr(self):
        """(row_ptr, col, val) of A as stored on the device."""
        rp = np.zeros(self._m + 1, np.int64)
        ci = np.zeros(max(self._nnz, 1), np.int32)
        va = np.zeros(max(self._nnz, 1), np.float64)
        _check(L.load().equil_matrix_export_csr(self._h, L.ptr(rp, L._i64p), L.ptr(ci, L._i32p),
                                                L.ptr(va, L._dp)))
        return rp, ci[: self._nnz], va[: self._nnz]

    def to_dense(self):
        """Row-major values of a dense matrix."""
        a = np.zeros((self._m, self._n))
        _check(L.load().equil_matrix_export_dense(self._h, L.ptr(a, L._dp)))
        return a

    def close(self):
        if self._h is not None and self._h.value:
            L.load().equil_matrix_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- LinearOperator ----------------------------------------------------
    def rows(self) -> int:
        return self._m

    def cols(self) -> int:
        return self._n

    def is_sparse(self) -> bool:
        return not self._dense

    def stored_entries(self) -> int:
        return self._nnz

    def apply(self, x) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        if x.size != self._n:
            raise InvalidArgument("ExplicitMatrix::apply: size mismatch")
        y = np.zeros(self._m)
        _check(L.load().equil_apply(self._h, L.ptr(x, L._dp), L.ptr(y, L._dp), 0))
        return y

    def apply_adjoint(self, y) -> np.ndarray:
        y = np.ascontiguousarray(y, dtype=np.float64)
        if y.size != self._m:
            raise InvalidArgument("ExplicitMatrix::apply_adjoint: size mismatch")
        x = np.zeros(self._n)
        _check(L.load().equil_apply(self._h, L.ptr(y, L._dp), L.ptr(x, L._dp), 1))
        return x

    def transposed_csr(self):
        """CSR(A^T) exactly as built on the device (verification hook)."""
        trp = np.zeros(self._n + 1, np.int64)
        tc = np.zeros(max(self._nnz, 1), np.int32)
        tv = np.zeros(max(self._nnz, 1), np.float64)
        _check(L.load().equil_export_transpose(self._h, L.ptr(trp, L._i64p),
                                               L.ptr(tc, L._i32p), L.ptr(tv, L._dp)))
        return trp, tc[: self._nnz], tv[: self._nnz]


def sgd_equilibrate(op: ExplicitMatrix, params: EquilibrationParams | None = None,
                    diag: DiagnosticsConfig | None = None) -> ScalingResult:
    """sgd_equilibrate (include/equil/equilibrate.hpp:89-91)."""
    params = params or EquilibrationParams()
    m, n = op.rows(), op.cols()
    u, v, d, e = np.zeros(m), np.zeros(n), np.zeros(m), np.zeros(n)
    cap = (max(int(params.iterations), 0) // diag.stride + 1) if diag and diag.stride > 0 else 1
    hi = np.zeros(cap, np.int32)
    ho = np.zeros(cap)
    hr = np.zeros(cap)
    out = L.ScalingOut(L.ptr(u, L._dp), L.ptr(v, L._dp), L.ptr(d, L._dp), L.ptr(e, L._dp), 0,
                       0.0, 0.0, 0, 0, 0, 0, L.ptr(hi, L._ip), L.ptr(ho, L._dp),
                       L.ptr(hr, L._dp), cap, 0)
    p = params._c()
    dc = L.DiagCfg(diag.stride, int(diag.want_objective), int(diag.want_rms)) if diag else None
    _check(L.load().equil_sgd_equilibrate(op._h, C.byref(p),
                                          C.byref(dc) if dc is not None else None,
                                          C.byref(out)))
    hist = [IterationRecord(int(hi[k]), float(ho[k]) if diag.want_objective else None,
                            float(hr[k]) if diag.want_rms else None)
            for k in range(out.hist_len)] if diag else []
    return ScalingResult(u, v, d, e, out.alpha, out.beta, hist, bool(out.box_feasible),
                         bool(out.iterate_bound_ok), out.apply_count, out.adjoint_count)


class DeviceOperator:
    """A matrix-free LinearOperator on the device (include/equil/linop.hpp:13-25).

    apply(x_ptr, y_ptr, stream) must compute y = A x and apply_adjoint(y_ptr,
    x_ptr, stream) x = A^T y, on device pointers (ints) of cols / rows doubles,
    enqueued on the CUDA stream handle `stream` (or finished before returning).
    """

    def __init__(self, rows: int, cols: int, apply, apply_adjoint, device: int = 0):
        self.rows_, self.cols_, self.device = int(rows), int(cols), int(device)
        # keep the ctypes trampolines alive as long as the operator
        self._fa = L.DeviceApplyFn(lambda ctx, i, o, s: apply(i, o, s))
        self._fb = L.DeviceApplyFn(lambda ctx, i, o, s: apply_adjoint(i, o, s))

    @classmethod
    def from_matrix(cls, M: ExplicitMatrix, device: int = 0) -> "DeviceOperator":
        """An explicit matrix's own device apply / adjoint as an operator."""
        lib = L.load()
        return cls(M.rows(), M.cols(),
                   lambda x, y, s: _check(lib.equil_apply_device(M._h, x, y, 0, s)),
                   lambda y, x, s: _check(lib.equil_apply_device(M._h, y, x, 1, s)),
                   device=device)

    def rows(self) -> int:
        return self.rows_

    def cols(self) -> int:
        return self.cols_

    def _c(self):
        return L.DeviceOperator(self.rows_, self.cols_, self._fa, self._fb, None, self.device)


def sgd_equilibrate_operator(op: DeviceOperator,
                             params: EquilibrationParams | None = None) -> ScalingResult:
    """sgd_equilibrate (include/equil/equilibrate.hpp:89-91) on a matrix-free
    device operator: T applies and T adjoints of op, everything else on the
    device.  No history (the reference needs the explicit matrix for it)."""
    params = params or EquilibrationParams()
    m, n = op.rows(), op.cols()
    u, v, d, e = np.zeros(m), np.zeros(n), np.zeros(m), np.zeros(n)
    out = L.ScalingOut(L.ptr(u, L._dp), L.ptr(v, L._dp), L.ptr(d, L._dp), L.ptr(e, L._dp), 0,
                       0.0, 0.0, 0, 0, 0, 0, None, None, None, 0, 0)
    p = params._c()
    c_op = op._c()
    _check(L.load().equil_sgd_equilibrate_operator(C.byref(c_op), C.byref(p), C.byref(out)))
    return ScalingResult(u, v, d, e, out.alpha, out.beta, [], bool(out.box_feasible),
                         bool(out.iterate_bound_ok), out.apply_count, out.adjoint_count)


def lsqr_operator(op: DeviceOperator, b, max_iters: int, rel_residual_tol: float,
                  equil_params: EquilibrationParams | None = None) -> LsqrRun:
    """lsqr (equil_params None) or lsqr_preconditioned (include/equil/lsqr.hpp:
    30-40) on a matrix-free device operator."""
    b = np.ascontiguousarray(b, dtype=np.float64)
    who = "lsqr_preconditioned" if equil_params is not None else "lsqr"
    if b.size != op.rows():
        raise InvalidArgument(f"{who}: rhs length mismatch")
    x = np.zeros(op.cols())
    T = max(int(equil_params.iterations), 0) if equil_params is not None else 0
    h = np.zeros(max(max_iters, 0) + T + 2)
    out = L.LsqrOut(L.ptr(x, L._dp), L.ptr(h, L._dp), h.size, 0, 0, 0, 0, 0, 0, 0)
    p = equil_params._c() if equil_params is not None else None
    c_op = op._c()
    _check(L.load().equil_lsqr_operator(C.byref(c_op), L.ptr(b, L._dp),
                                        C.byref(p) if p is not None else None, int(max_iters),
                                        float(rel_residual_tol), C.byref(out)))
    return _lsqr_run(x, h, out)


def sgd_equilibrate_targets(op: ExplicitMatrix, r, c, params: EquilibrationParams | None = None,
                            diag: DiagnosticsConfig | None = None) -> ScalingResult:
    """sgd_equilibrate_targets (include/equil/variants.hpp:24-27): row i aims
    at squared norm r_i, column j at c_j; history carries the objective only
    (alpha/beta of the result are 0, as in the reference)."""
    params = params or EquilibrationParams()
    r = np.ascontiguousarray(r, dtype=np.float64)
    c = np.ascontiguousarray(c, dtype=np.float64)
    if r.size != op.rows() or c.size != op.cols():
        raise InvalidArgument("sgd_equilibrate_targets: target length mismatch")
    m, n = op.rows(), op.cols()
    u, v, d, e = np.zeros(m), np.zeros(n), np.zeros(m), np.zeros(n)
    cap = (max(int(params.iterations), 0) // diag.stride + 1) if diag and diag.stride > 0 else 1
    hi, ho, hr = np.zeros(cap, np.int32), np.zeros(cap), np.zeros(cap)
    out = L.ScalingOut(L.ptr(u, L._dp), L.ptr(v, L._dp), L.ptr(d, L._dp), L.ptr(e, L._dp), 0,
                       0.0, 0.0, 0, 0, 0, 0, L.ptr(hi, L._ip), L.ptr(ho, L._dp),
                       L.ptr(hr, L._dp), cap, 0)
    p = params._c()
    dc = L.DiagCfg(diag.stride, int(diag.want_objective), 0) if diag else None
    _check(L.load().equil_sgd_equilibrate_targets(op._h, L.ptr(r, L._dp), L.ptr(c, L._dp),
                                                  C.byref(p),
                                                  C.byref(dc) if dc is not None else None,
                                                  C.byref(out)))
    hist = [IterationRecord(int(hi[k]), float(ho[k]) if diag.want_objective else None, None)
            for k in range(out.hist_len)] if diag else []
    return ScalingResult(u, v, d, e, out.alpha, out.beta, hist, bool(out.box_feasible),
                         bool(out.iterate_bound_ok), out.apply_count, out.adjoint_count)


@dataclass
class BlockStructure:
    """BlockStructure (include/equil/variants.hpp:30-39): row i belongs to row
    block row_block[i], column j to column block col_block[j]."""
    row_block: np.ndarray
    col_block: np.ndarray
    row_blocks: int
    col_blocks: int

    @staticmethod
    def trivial(rows: int, cols: int) -> "BlockStructure":
        """One row (column) per block (src/variants.cpp:120-129)."""
        return BlockStructure(np.arange(rows, dtype=np.int64), np.arange(cols, dtype=np.int64),
                              int(rows), int(cols))


def _variant_call(op, params, diag, call):
    m, n = op.rows(), op.cols()
    u, v, d, e = np.zeros(m), np.zeros(n), np.zeros(m), np.zeros(n)
    cap = (max(int(params.iterations), 0) // diag.stride + 1) if diag and diag.stride > 0 else 1
    hi, ho, hr = np.zeros(cap, np.int32), np.zeros(cap), np.zeros(cap)
    out = L.ScalingOut(L.ptr(u, L._dp), L.ptr(v, L._dp), L.ptr(d, L._dp), L.ptr(e, L._dp), 0,
                       0.0, 0.0, 0, 0, 0, 0, L.ptr(hi, L._ip), L.ptr(ho, L._dp),
                       L.ptr(hr, L._dp), cap, 0)
    p = params._c()
    dc = L.DiagCfg(diag.stride, int(diag.want_objective), int(diag.want_rms)) if diag else None
    _check(call(C.byref(p), C.byref(dc) if dc is not None else None, C.byref(out)))
    hist = [IterationRecord(int(hi[k]), float(ho[k]) if diag.want_objective else None,
                            float(hr[k]) if diag.want_rms else None)
            for k in range(out.hist_len)] if diag else []
    return ScalingResult(u, v, d, e, out.alpha, out.beta, hist, bool(out.box_feasible),
                         bool(out.iterate_bound_ok), out.apply_count, out.adjoint_count)


def sgd_equilibrate_symmetric(op: ExplicitMatrix, params: EquilibrationParams | None = None,
                              diag: DiagnosticsConfig | None = None) -> ScalingResult:
    """sgd_equilibrate_symmetric (include/equil/variants.hpp:16-18): one
    scaling on both sides of a symmetric matrix; u == v and d == e."""
    params = params or EquilibrationParams()
    return _variant_call(op, params, diag, lambda p, dc, out: L.load()
                         .equil_sgd_equilibrate_symmetric(op._h, p, dc, out))


def sgd_equilibrate_block(op: ExplicitMatrix, structure: BlockStructure,
                          params: EquilibrationParams | None = None,
                          diag: DiagnosticsConfig | None = None) -> ScalingResult:
    """sgd_equilibrate_block (include/equil/variants.hpp:47-50): rows (columns)
    of one block share a scaling; results expanded to full length."""
    params = params or EquilibrationParams()
    rb = np.ascontiguousarray(structure.row_block, dtype=np.int64)
    cb = np.ascontiguousarray(structure.col_block, dtype=np.int64)
    if rb.size != op.rows() or cb.size != op.cols():
        raise InvalidArgument("BlockStructure: assignment length mismatch")
    return _variant_call(op, params, diag, lambda p, dc, out: L.load()
                         .equil_sgd_equilibrate_block(op._h, L.ptr(rb, L._i64p),
                                                      L.ptr(cb, L._i64p),
                                                      int(structure.row_blocks),
                                                      int(structure.col_blocks), p, dc, out))


@dataclass
class LassoProblem:
    """LassoProblem (include/equil/ccp.hpp:14-18): min |A x - b|^2 / sqrt(lambda)
    + sqrt(lambda) |x|_1."""
    op: ExplicitMatrix
    b: np.ndarray
    lam: float


@dataclass
class CcpOptions:
    """CcpOptions (include/equil/ccp.hpp:24-33)."""
    max_iters: int = 1000
    tau: float = 0.0     # 0 = auto 0.9 / |K|_2
    sigma: float = 0.0
    theta: float = 1.0
    p_star: float = float("nan")  # NaN disables gap_history
    gap_tol: float = 0.0


@dataclass
class CcpRun:
    """CcpRun (include/equil/ccp.hpp:35-48)."""
    x: np.ndarray
    objective_history: list
    gap_history: list
    tau: float
    sigma: float
    theta: float
    iterations: int
    equil_iterations: int
    reached_tol: bool
    apply_count: int
    adjoint_count: int


def _ccp(prob: LassoProblem, params, options: CcpOptions | None) -> CcpRun:
    options = options or CcpOptions()
    b = np.ascontiguousarray(prob.b, dtype=np.float64)
    if b.size != prob.op.rows():
        raise InvalidArgument("lasso: rhs length mismatch")
    T = max(int(params.iterations), 0) if params is not None else 0
    cap = max(int(options.max_iters), 0) + 1 + T
    x, oh, gh = np.zeros(prob.op.cols()), np.zeros(cap), np.zeros(cap)
    o = L.CcpOptions(int(options.max_iters), float(options.tau), float(options.sigma),
                     float(options.theta), float(options.p_star), float(options.gap_tol))
    out = L.CcpOut(L.ptr(x, L._dp), L.ptr(oh, L._dp), L.ptr(gh, L._dp), cap, 0, 0, 0.0, 0.0,
                   0.0, 0, 0, 0, 0, 0)
    lib = L.load()
    if params is None:
        _check(lib.equil_ccp_lasso(prob.op._h, L.ptr(b, L._dp), float(prob.lam), C.byref(o),
                                   C.byref(out)))
    else:
        p = params._c()
        _check(lib.equil_ccp_lasso_preconditioned(prob.op._h, L.ptr(b, L._dp), float(prob.lam),
                                                  C.byref(p), C.byref(o), C.byref(out)))
    return CcpRun(x, oh[:out.hist_len].tolist(), gh[:out.gap_len].tolist(), out.tau, out.sigma,
                  out.theta, out.iterations, out.equil_iterations, bool(out.reached_tol),
                  out.apply_count, out.adjoint_count)


def ccp_lasso(prob: LassoProblem, options: CcpOptions | None = None) -> CcpRun:
    """ccp_lasso (include/equil/ccp.hpp:57, src/ccp.cpp:125-132)."""
    return _ccp(prob, None, options)


def ccp_lasso_preconditioned(prob: LassoProblem, params: EquilibrationParams,
                             options: CcpOptions | None = None) -> CcpRun:
    """ccp_lasso_preconditioned (include/equil/ccp.hpp:65-67, src/ccp.cpp:134-141)."""
    return _ccp(prob, params, options)


def spectral_norm(op: ExplicitMatrix, max_iters: int = 100, rel_tol: float = 1e-6,
                  seed: int = 0) -> float:
    """spectral_norm (include/equil/lsqr.hpp:44-48, src/lsqr.cpp:140-163)."""
    out = C.c_double(0.0)
    _check(L.load().equil_spectral_norm(op._h, int(max_iters), float(rel_tol), int(seed),
                                        C.byref(out)))
    return out.value


def lasso_objective(prob: LassoProblem, x) -> float:
    """lasso_objective (include/equil/ccp.hpp:21, src/ccp.cpp:115-123)."""
    b = np.ascontiguousarray(prob.b, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64)
    if x.size != prob.op.cols():
        raise InvalidArgument("lasso_objective: x length mismatch")
    out = C.c_double(0.0)
    _check(L.load().equil_lasso_objective(prob.op._h, L.ptr(b, L._dp), float(prob.lam),
                                          L.ptr(x, L._dp), C.byref(out)))
    return out.value


@dataclass
class MatrixMarketData:
    """A parsed Matrix Market file on the host (no device involved)."""
    m: int
    n: int
    dense: bool
    rows: np.ndarray   # 0-based, file order (coordinate)
    cols: np.ndarray
    vals: np.ndarray   # coordinate values, or row-major m x n (array)
    lines: np.ndarray  # line number of every coordinate entry


def parse_matrix_market(path: str) -> MatrixMarketData:
    """The host half of read_matrix_market (src/matrix_market.cpp:63-198):
    header / size / entry rules and their line-numbered errors.  Duplicate
    detection happens with the device sort in ExplicitMatrix.read_matrix_market."""
    lib = L.load()
    m, n, nnz, dn = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int()
    h = C.c_void_p()
    _check(lib.equil_mm_parse(str(path).encode(), C.byref(m), C.byref(n), C.byref(nnz),
                              C.byref(dn), C.byref(h)))
    try:
        if dn.value:
            v = np.zeros((m.value, n.value))
            _check(lib.equil_mm_fetch(h, None, None, L.ptr(v, L._dp), None))
            z = np.zeros(0, np.int64)
            return MatrixMarketData(m.value, n.value, True, z, z, v, z)
        k = nnz.value
        r, c, ln = (np.zeros(max(k, 1), np.int64) for _ in range(3))
        v = np.zeros(max(k, 1))
        _check(lib.equil_mm_fetch(h, L.ptr(r, L._i64p), L.ptr(c, L._i64p), L.ptr(v, L._dp),
                                  L.ptr(ln, L._i64p)))
        return MatrixMarketData(m.value, n.value, False, r[:k], c[:k], v[:k], ln[:k])
    finally:
        lib.equil_mm_free(h)


def write_matrix_market_csr(path: str, m: int, n: int, row_ptr, col, val):
    """write_matrix_market (src/matrix_market.cpp:209-233) of a host CSR."""
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(col, dtype=np.int32)
    va = np.ascontiguousarray(val, dtype=np.float64)
    _check(L.load().equil_mm_write_csr(str(path).encode(), m, n, L.ptr(rp, L._i64p),
                                       L.ptr(ci, L._i32p), L.ptr(va, L._dp)))


def write_matrix_market_dense(path: str, values):
    a = np.ascontiguousarray(values, dtype=np.float64)
    _check(L.load().equil_mm_write_dense(str(path).encode(), a.shape[0], a.shape[1],
                                         L.ptr(a, L._dp)))


class SeededRng:
    """SeededRng (include/equil/rng.hpp:12-42) as a position in the (seed,
    stream) output sequence; consumers advance it by the draws they use."""

    def __init__(self, seed: int, stream: int):
        self.seed, self.stream, self.position = int(seed), int(stream), 0


def _vecs(op, u, v):
    u = np.ascontiguousarray(u, dtype=np.float64)
    v = np.ascontiguousarray(v, dtype=np.float64)
    if u.size != op.rows() or v.size != op.cols():
        raise InvalidArgument("objective: scaling length mismatch")
    return u, v


def objective(op: ExplicitMatrix, u, v, params: EquilibrationParams | None = None) -> float:
    """objective (include/equil/equilibrate.hpp:23-24)."""
    u, v = _vecs(op, u, v)
    p = (params or EquilibrationParams())._c()
    out = C.c_double(0.0)
    _check(L.load().equil_objective(op._h, L.ptr(u, L._dp), L.ptr(v, L._dp), C.byref(p),
                                    C.byref(out)))
    return out.value


def objective_weighted(op: ExplicitMatrix, u, v, lin_u, lin_v, gamma: float) -> float:
    """objective_weighted (include/equil/equilibrate.hpp:35-36)."""
    u, v = _vecs(op, u, v)
    lu = np.ascontiguousarray(lin_u, dtype=np.float64)
    lv = np.ascontiguousarray(lin_v, dtype=np.float64)
    out = C.c_double(0.0)
    _check(L.load().equil_objective_weighted(op._h, L.ptr(u, L._dp), L.ptr(v, L._dp),
                                             L.ptr(lu, L._dp), L.ptr(lv, L._dp), float(gamma),
                                             C.byref(out)))
    return out.value


def gradient(op: ExplicitMatrix, u, v, params: EquilibrationParams | None = None):
    """gradient (include/equil/equilibrate.hpp:29-30) -> (grad_u, grad_v)."""
    u, v = _vecs(op, u, v)
    p = (params or EquilibrationParams())._c()
    gu, gv = np.zeros(op.rows()), np.zeros(op.cols())
    _check(L.load().equil_gradient(op._h, L.ptr(u, L._dp), L.ptr(v, L._dp), C.byref(p),
                                   L.ptr(gu, L._dp), L.ptr(gv, L._dp)))
    return gu, gv


def gradient_weighted(op: ExplicitMatrix, u, v, lin_u, lin_v, gamma: float):
    """gradient_weighted (include/equil/equilibrate.hpp:37-39)."""
    u, v = _vecs(op, u, v)
    lu = np.ascontiguousarray(lin_u, dtype=np.float64)
    lv = np.ascontiguousarray(lin_v, dtype=np.float64)
    gu, gv = np.zeros(op.rows()), np.zeros(op.cols())
    _check(L.load().equil_gradient_weighted(op._h, L.ptr(u, L._dp), L.ptr(v, L._dp),
                                            L.ptr(lu, L._dp), L.ptr(lv, L._dp), float(gamma),
                                            L.ptr(gu, L._dp), L.ptr(gv, L._dp)))
    return gu, gv


def stochastic_gradient_estimate(op: ExplicitMatrix, u, v, params: EquilibrationParams,
                                 rng: SeededRng):
    """stochastic_gradient_estimate (include/equil/equilibrate.hpp:43-45):
    consumes n + m draws of rng (s for the apply, then w for the adjoint)."""
    u, v = _vecs(op, u, v)
    p = params._c()
    gu, gv = np.zeros(op.rows()), np.zeros(op.cols())
    _check(L.load().equil_stochastic_gradient_estimate(
        op._h, L.ptr(u, L._dp), L.ptr(v, L._dp), C.byref(p), rng.seed, rng.stream,
        rng.position, L.ptr(gu, L._dp), L.ptr(gv, L._dp)))
    rng.position += op.rows() + op.cols()
    return gu, gv


def rms_error(op: ExplicitMatrix, u, v, alpha: float, beta: float) -> float:
    """rms_error (include/equil/metrics.hpp:14-15)."""
    u, v = _vecs(op, u, v)
    out = C.c_double(0.0)
    _check(L.load().equil_rms_error(op._h, L.ptr(u, L._dp), L.ptr(v, L._dp), float(alpha),
                                    float(beta), C.byref(out)))
    return out.value


def project_box(x, bound: float) -> np.ndarray:
    """project_box (include/equil/equilibrate.hpp:48)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.zeros_like(x)
    _check(L.load().equil_project_box(L.ptr(x, L._dp), x.size, float(bound), L.ptr(out, L._dp)))
    return out


def sgd_equilibrate_device(op: ExplicitMatrix, params: EquilibrationParams,
                           u_ptr: int, v_ptr: int, d_ptr: int, e_ptr: int) -> ScalingResult:
    """sgd_equilibrate with u, v, d, e written to caller-owned DEVICE buffers
    (raw pointers, e.g. torch tensors' data_ptr()); the vectors in the returned
    record are empty."""
    p = params._c()
    dp = C.POINTER(C.c_double)
    out = L.ScalingOut(C.cast(u_ptr, dp), C.cast(v_ptr, dp), C.cast(d_ptr, dp),
                       C.cast(e_ptr, dp), 1, 0.0, 0.0, 0, 0, 0, 0, None, None, None, 0, 0)
    _check(L.load().equil_sgd_equilibrate(op._h, C.byref(p), None, C.byref(out)))
    z = np.zeros(0)
    return ScalingResult(z, z, z, z, out.alpha, out.beta, [], bool(out.box_feasible),
                         bool(out.iterate_bound_ok), out.apply_count, out.adjoint_count)


def sgd_equilibrate_csr(rows: int, cols: int, row_ptr, col, val,
                        params: EquilibrationParams, device: int = 0,
                        out=None) -> ScalingResult:
    """One-shot C-ABI entry (equil_sgd_equilibrate_csr): host CSR in, host
    scaling out; upload, device transpose, equilibration and download inside.
    out: optional (u, v, d, e) float64 host arrays (e.g. pinned) to write into."""
    if out is None:
        u, v, d, e = np.zeros(rows), np.zeros(cols), np.zeros(rows), np.zeros(cols)
    else:
        u, v, d, e = out
        for a, ln in ((u, rows), (v, cols), (d, rows), (e, cols)):
            if a.dtype != np.float64 or a.shape != (ln,) or not a.flags.c_contiguous:
                raise ValueError("sgd_equilibrate_csr: out arrays must be contiguous float64 "
                                 "of lengths (rows, cols, rows, cols)")
    out = L.ScalingOut(L.ptr(u, L._dp), L.ptr(v, L._dp), L.ptr(d, L._dp), L.ptr(e, L._dp), 0,
                       0.0, 0.0, 0, 0, 0, 0, None, None, None, 0, 0)
    p = params._c()
    cfg = L.DeviceCfg(device, 0, 1, None)
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    _check(L.load().equil_sgd_equilibrate_csr(
        rows, cols, L.ptr(rp, L._i64p), col.ctypes.data_as(L._i32p),
        val.ctypes.data_as(L._dp), C.byref(p), C.byref(cfg), C.byref(out)))
    return ScalingResult(u, v, d, e, out.alpha, out.beta, [], bool(out.box_feasible),
                         bool(out.iterate_bound_ok), out.apply_count, out.adjoint_count)


def last_loop_ms(op: ExplicitMatrix):
    """(device ms of the last call's T-iteration loop, T)"""
    it = C.c_int()
    ms = L.load().equil_last_loop_ms(op._h, C.byref(it))
    return ms, it.value


def exchange_mode(op: ExplicitMatrix) -> str:
    """How a sharded handle's SGD loop exchanges the gathered vectors:
    "single" (one GPU or not yet run), "allgather" or "p2p" (fused peer stores)."""
    return ("single", "allgather", "p2p")[int(L.load().equil_exchange_mode(op._h))]


def sweep_active(op: ExplicitMatrix) -> bool:
    """True if the SGD passes run A's rows of more than 512 entries on the
    column sweep (csrc/sweep.cu) rather than the long-slice kernel."""
    return bool(L.load().equil_sweep_active(op._h))


def kernel_launches() -> int:
    return int(L.load().equil_kernel_launches())


def _lsqr_run(x, h, out) -> LsqrRun:
    return LsqrRun(x, list(h[: out.hist_len]), out.iterations, out.equil_iterations,
                   bool(out.reached_tol), bool(out.breakdown), out.apply_count,
                   out.adjoint_count)


def lsqr(op: ExplicitMatrix, b, max_iters: int, rel_residual_tol: float) -> LsqrRun:
    """lsqr (include/equil/lsqr.hpp:30-31)."""
    b = np.ascontiguousarray(b, dtype=np.float64)
    if b.size != op.rows():
        raise InvalidArgument("lsqr: rhs length mismatch")
    x = np.zeros(op.cols())
    h = np.zeros(max(max_iters, 0) + 1)
    out = L.LsqrOut(L.ptr(x, L._dp), L.ptr(h, L._dp), h.size, 0, 0, 0, 0, 0, 0, 0)
    _check(L.load().equil_lsqr(op._h, L.ptr(b, L._dp), int(max_iters), float(rel_residual_tol),
                               C.byref(out)))
    return _lsqr_run(x, h, out)


def lsqr_preconditioned(op: ExplicitMatrix, b, equil_params: EquilibrationParams,
                        max_iters: int, rel_residual_tol: float) -> LsqrRun:
    """lsqr_preconditioned (include/equil/lsqr.hpp:38-40)."""
    b = np.ascontiguousarray(b, dtype=np.float64)
    if b.size != op.rows():
        raise InvalidArgument("lsqr_preconditioned: rhs length mismatch")
    x = np.zeros(op.cols())
    h = np.zeros(max(max_iters, 0) + max(int(equil_params.iterations), 0) + 2)
    out = L.LsqrOut(L.ptr(x, L._dp), L.ptr(h, L._dp), h.size, 0, 0, 0, 0, 0, 0, 0)
    p = equil_params._c()
    _check(L.load().equil_lsqr_preconditioned(op._h, L.ptr(b, L._dp), C.byref(p),
                                              int(max_iters), float(rel_residual_tol),
                                              C.byref(out)))
    return _lsqr_run(x, h, out)


def sign_bits(seed: int, stream: int, start: int, count: int, device: int = 0) -> np.ndarray:
    """Device-generated probe sign bits (verification hook, K1)."""
    out = np.zeros((count + 31) // 32 + 1, np.uint32)
    _check(L.load().equil_sign_bits(seed, stream, start, count, L.ptr(out, L._u32p), device))
    return out[: (count + 31) // 32]


def det_exp_device(x, device: int = 0) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.zeros_like(x)
    _check(L.load().equil_det_exp_device(L.ptr(x, L._dp), L.ptr(y, L._dp), x.size, device))
    return y


def canon_sumsq_device(x, device: int = 0) -> float:
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = C.c_double()
    _check(L.load().equil_canon_sumsq_device(L.ptr(x, L._dp), x.size, C.byref(out), device))
    return out.value


def partition_rows(row_ptr, parts: int) -> np.ndarray:
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    b = np.zeros(parts + 1, np.int64)
    _check(L.load().equil_partition_rows(L.ptr(rp, L._i64p), rp.size - 1, parts,
                                         L.ptr(b, L._i64p)))
    return b


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(L.load().equil_nccl_unique_id(buf))
    return buf.raw
