"""Seeded synthetic instances for BASELINE.json's five configs.

There is no public dataset for this path; these restate the
config text.  Interpretation choices:
  * N(0, s) means standard deviation s;
  * config 1 has exactly n * 1% = 50 distinct uniform columns per row;
  * config 3 keeps the stated generator (Zipf exponent 1.5 on [1, 10^4]), which
    gives nnz ~ 1.53e8 rather than the text's "~5e7";
  * config 5 row lengths are round(LogNormal(ln 50 - 1/2, 1)) clamped to [1, n].
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass

import numpy as np

from . import build as _build

_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)
_gen = None


def _lib():
    global _gen
    if _gen is None:
        if not os.path.exists(_build.GEN_LIB):
            _build.build()
        g = C.CDLL(_build.GEN_LIB)
        g.gen_row_ptr.restype = C.c_int64
        g.gen_row_ptr.argtypes = [C.c_int64, C.c_int64, C.c_int, C.c_double, C.c_double,
                                  C.c_uint64, _i64p]
        g.gen_fill.argtypes = [C.c_int64, C.c_int64, _i64p, C.c_uint64, C.c_double,
                               C.c_double, _i32p, _dp]
        g.gen_dense.argtypes = [C.c_int64, C.c_int64, C.c_uint64, C.c_double, C.c_double, _dp]
        g.gen_normal.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, _dp]
        _gen = g
    return _gen


@dataclass
class Instance:
    name: str
    m: int
    n: int
    row_ptr: np.ndarray | None = None
    col: np.ndarray | None = None
    val: np.ndarray | None = None
    dense: np.ndarray | None = None
    alpha: float = 0.0
    beta: float = 0.0
    iterations: int = 100
    seed: int = 0

    @property
    def nnz(self) -> int:
        return self.m * self.n if self.dense is not None else int(self.row_ptr[-1])


def sparse(m, n, kind, p0, p1, seed, sr, sc, pinned_alloc=None) -> tuple:
    g = _lib()
    rp = np.zeros(m + 1, np.int64)
    nnz = g.gen_row_ptr(m, n, kind, p0, p1, seed, rp.ctypes.data_as(_i64p))
    if pinned_alloc is not None:
        col, val = pinned_alloc(nnz)
    else:
        col, val = np.empty(nnz, np.int32), np.empty(nnz, np.float64)
    g.gen_fill(m, n, rp.ctypes.data_as(_i64p), seed, sr, sc, col.ctypes.data_as(_i32p),
               val.ctypes.data_as(_dp))
    return rp, col, val


def dense(m, n, seed, sr, sc) -> np.ndarray:
    a = np.empty((m, n), np.float64)
    _lib().gen_dense(m, n, seed, sr, sc, a.ctypes.data_as(_dp))
    return a


def normal(seed, stream, count) -> np.ndarray:
    out = np.empty(count, np.float64)
    _lib().gen_normal(seed, stream, count, out.ctypes.data_as(_dp))
    return out


def config(k: int, scale: float = 1.0, pinned_alloc=None) -> Instance:
    """BASELINE.json configs[k-1]; ``scale`` shrinks m, n (tests)."""
    if k == 1:
        m, n = int(10000 * scale), int(5000 * scale)
        rp, c, v = sparse(m, n, 0, max(1, round(0.01 * n)), 0, 101, 1.0, 1.0, pinned_alloc)
        return Instance("c1 sparse 10000x5000 1% fp64", m, n, rp, c, v, alpha=math.sqrt(n / m),
                        beta=1.0, iterations=50, seed=0)
    if k == 2:
        m, n = int(4096 * scale), int(2048 * scale)
        a = dense(m, n, 202, 2.0, 2.0)
        return Instance("c2 dense 4096x2048 fp64", m, n, dense=a, iterations=100, seed=1)
    if k in (3, 4):
        m, n = int(2_000_000 * scale), int(1_000_000 * scale)
        rp, c, v = sparse(m, n, 1, 1.5, min(10_000, n), 303, 1.5, 1.5, pinned_alloc)
        return Instance("c3 sparse 2e6x1e6 zipf1.5 fp64" if k == 3 else "c4 lsqr on c3",
                        m, n, rp, c, v, iterations=100 if k == 3 else 50, seed=0)
    if k == 5:
        m, n = int(20_000_000 * scale), int(10_000_000 * scale)
        rp, c, v = sparse(m, n, 2, math.log(50) - 0.5, 1.0, 505, 2.0, 2.0, pinned_alloc)
        return Instance("c5 sparse 2e7x1e7 lognormal fp64", m, n, rp, c, v, iterations=100,
                        seed=0)
    raise ValueError(k)


def rhs(inst: Instance, seed: int = 404) -> np.ndarray:
    """Config 4: b = A x_true + 0.01 N(0,1), x_true ~ N(0,1)."""
    x = normal(seed, 0, inst.n)
    noise = normal(seed, 1, inst.m)
    if inst.dense is not None:
        ax = inst.dense @ x
    else:
        rows = np.repeat(np.arange(inst.m), np.diff(inst.row_ptr))
        ax = np.bincount(rows, weights=inst.val * x[inst.col], minlength=inst.m)
    return ax + 0.01 * noise
