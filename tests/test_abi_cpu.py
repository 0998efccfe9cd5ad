"""CPU tests of the C ABI boundary (no compute calls need a GPU here)."""
import ctypes
import math
import os
import re

import numpy as np
import pytest

import paper_1602_06621_b200 as eq
from paper_1602_06621_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "equil_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(equil_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_reference_entry_points():
    names = declared_functions()
    for must in ["equil_sgd_equilibrate", "equil_lsqr", "equil_lsqr_preconditioned",
                 "equil_matrix_create_csr", "equil_matrix_create_dense", "equil_apply",
                 "equil_resolve_targets", "equil_validate_params", "equil_last_error"]:
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    # and the Python binding knows every one of them
    assert set(declared_functions()) <= set(_lib.SIGNATURES)


def test_det_exp_host_equals_oracle(C):
    L = _lib.load()
    rng = np.random.default_rng(5)
    xs = np.concatenate([rng.uniform(-20, 20, 20000), [0.0, -0.0, 9.210340371976184]])
    for x in xs:
        a = L.equil_det_exp_host(float(x))
        b = C.L.eo_det_exp(float(x))
        assert a == b or (math.isnan(a) and math.isnan(b))


def test_params_resolution_matches_reference_rules():
    # src/params.cpp:7-33
    a, b = eq.resolve_targets(eq.EquilibrationParams(), 10000, 5000)
    assert a == pytest.approx((5000 / 10000) ** 0.25, rel=0) and b == (10000 / 5000) ** 0.25
    a, b = eq.resolve_targets(eq.EquilibrationParams(alpha=2.0), 4, 1)
    assert (a, b) == (2.0, 2.0 * math.sqrt(4 / 1))
    a, b = eq.resolve_targets(eq.EquilibrationParams(beta=1.0), 10000, 5000)
    assert b == 1.0 and a == 1.0 * math.sqrt(5000 / 10000)
    with pytest.raises(eq.InvalidArgument, match="violated"):
        eq.resolve_targets(eq.EquilibrationParams(alpha=1.0, beta=1.0), 4, 1)
    with pytest.raises(eq.InvalidArgument, match="positive"):
        eq.resolve_targets(eq.EquilibrationParams(alpha=-1.0), 4, 1)
    with pytest.raises(eq.InvalidArgument, match="dimensions"):
        eq.resolve_targets(eq.EquilibrationParams(), 0, 1)
    eq.validate_params(eq.EquilibrationParams())
    for bad in [dict(gamma=0.0), dict(max_log_scale=-1.0), dict(iterations=-1),
                dict(gamma=float("inf"))]:
        with pytest.raises(eq.InvalidArgument):
            eq.validate_params(eq.EquilibrationParams(**bad))


def test_resolve_targets_matches_oracle(C):
    import oracle
    for m, n, al, be in [(10000, 5000, 0, 0), (7, 3, 0.5, 0), (3, 7, 0, 2.0)]:
        p = oracle._Params(al, be, 0.1, 9.2, 1, 0)
        a1, b1 = ctypes.c_double(), ctypes.c_double()
        C.L.eo_resolve_targets(ctypes.byref(p), m, n, ctypes.byref(a1), ctypes.byref(b1))
        a2, b2 = eq.resolve_targets(eq.EquilibrationParams(alpha=al, beta=be), m, n)
        assert (a1.value, b1.value) == (a2, b2)


def test_partition_rows_balances_and_covers():
    rng = np.random.default_rng(1)
    lens = rng.zipf(1.5, 10000).clip(1, 5000)
    rp = np.concatenate([[0], np.cumsum(lens)])
    for parts in [1, 2, 3, 8]:
        b = eq.partition_rows(rp, parts)
        assert b[0] == 0 and b[-1] == 10000 and np.all(np.diff(b) >= 0)
        cost = [rp[b[g + 1]] - rp[b[g]] + b[g + 1] - b[g] for g in range(parts)]
        assert max(cost) <= (rp[-1] + 10000) / parts + lens.max() + 1


def test_product_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(eq.EquilRuntimeError):
        eq.ExplicitMatrix.identity(3)


def test_host_side_preconditions_need_no_gpu():
    # checks that precede any device work (src/explicit_matrix.cpp:21-22)
    with pytest.raises(eq.InvalidArgument, match="dimensions"):
        eq.ExplicitMatrix.sparse(0, 2, [])
    with pytest.raises(eq.InvalidArgument, match="row_ptr"):
        eq.ExplicitMatrix.from_csr(2, 2, [0, 2, 1], [0, 1], [1.0, 1.0])


def test_one_shot_result_buffers_are_checked_before_any_device_work():
    # sgd_equilibrate_csr(out=...): caller-owned (e.g. pinned) result arrays must
    # be contiguous float64 of lengths (rows, cols, rows, cols)
    import numpy as np
    rp = np.array([0, 1, 2], np.int64)
    col = np.array([0, 1], np.int32)
    val = np.array([1.0, 2.0])
    p = eq.EquilibrationParams(iterations=1)
    bad = [(np.zeros(2), np.zeros(2), np.zeros(2), np.zeros(3)),
           (np.zeros(2, np.float32), np.zeros(2), np.zeros(2), np.zeros(2)),
           (np.zeros(4)[::2], np.zeros(2), np.zeros(2), np.zeros(2))]
    for out in bad:
        with pytest.raises(ValueError, match="out arrays"):
            eq.sgd_equilibrate_csr(2, 2, rp, col, val, p, out=out)
