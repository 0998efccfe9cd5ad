"""The column sweep of A's long rows (csrc/sweep.cu): bit-exact
against the oracle and against the long-slice kernel (EQUIL_SWEEP=0), for the
default panel width, narrow panels (many panels, a partial last panel, three
stages) and the cases where the sweep must stand down (odd n, long rows in
A^T).  The knobs are read when a matrix handle is created."""
import os

import numpy as np
import pytest

import oracle  # checker
import paper_1602_06621_b200 as eq
from paper_1602_06621_b200 import configs

pytestmark = pytest.mark.gpu


def _with_env(env, fn):
    saved = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return fn()
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _run(inst, env, T=12, seed=5):
    def go():
        M = eq.ExplicitMatrix.from_csr(inst.m, inst.n, inst.row_ptr, inst.col, inst.val)
        r = eq.sgd_equilibrate(M, eq.EquilibrationParams(iterations=T, seed=seed))
        on = eq.sweep_active(M)
        M.close()
        return r, on
    return _with_env(env, go)


@pytest.fixture(scope="module")
def c3s():
    return configs.config(3, scale=0.02)  # 40000 x 20000, Zipf rows up to 10^4 entries


@pytest.mark.parametrize("env", [{}, {"EQUIL_SWEEP_WIDTH": "256", "EQUIL_SWEEP_STAGES": "3"},
                                 {"EQUIL_SWEEP_WIDTH": "1000"}, {"EQUIL_SWEEP_WIDTH": "20000"}],
                         ids=["default", "w256x3", "w1000", "one_panel"])
def test_sweep_bit_identical_to_oracle_and_long_kernel(c3s, env):
    inst = c3s
    A = oracle.CsrArrays(inst.m, inst.n, inst.row_ptr, inst.col, inst.val)
    want = oracle.c_oracle().sgd_equilibrate(A, iterations=12, seed=5)
    got, on = _run(inst, dict(env, EQUIL_SWEEP="1"))
    assert on, "the sweep did not engage on a matrix with long rows"
    base, off = _run(inst, {"EQUIL_SWEEP": "0"})
    assert not off
    for k in "uvde":
        assert np.array_equal(getattr(got, k), getattr(want, k)), k
        assert np.array_equal(getattr(got, k), getattr(base, k)), k


def test_sweep_is_default_for_handles_and_lsqr_unchanged(c3s):
    inst = c3s
    M = eq.ExplicitMatrix.from_csr(inst.m, inst.n, inst.row_ptr, inst.col, inst.val)
    assert eq.sweep_active(M)
    A = oracle.CsrArrays(inst.m, inst.n, inst.row_ptr, inst.col, inst.val)
    b = np.random.default_rng(3).standard_normal(inst.m)
    got = eq.lsqr_preconditioned(M, b, eq.EquilibrationParams(iterations=6, seed=2), 8, 0.0)
    want = oracle.c_oracle().lsqr_preconditioned(A, b, 8, 0.0, iterations=6, seed=2)
    assert np.array_equal(got.residual_history, want.residual_history)
    assert np.array_equal(got.x, want.x)
    M.close()


def _csr_from_rows(m, n, rows):
    rp = np.zeros(m + 1, dtype=np.int64)
    cols, vals = [], []
    for i, (c, v) in enumerate(rows):
        rp[i + 1] = rp[i] + len(c)
        cols.append(c)
        vals.append(v)
    return rp, np.concatenate(cols).astype(np.int32), np.concatenate(vals)


def test_sweep_stands_down(c3s):
    rng = np.random.default_rng(11)
    # odd n: the second xs buffer is not 16-byte aligned
    m, n = 300, 2001
    rows = []
    for i in range(m):
        L = 700 if i % 50 == 0 else int(rng.integers(1, 30))
        c = np.sort(rng.choice(n, size=L, replace=False))
        rows.append((c, rng.standard_normal(L)))
    rp, ci, va = _csr_from_rows(m, n, rows)
    M = eq.ExplicitMatrix.from_csr(m, n, rp, ci, va)
    assert not eq.sweep_active(M)
    r = eq.sgd_equilibrate(M, eq.EquilibrationParams(iterations=6, seed=1))
    w = oracle.c_oracle().sgd_equilibrate(oracle.CsrArrays(m, n, rp, ci, va), iterations=6, seed=1)
    for k in "uvde":
        assert np.array_equal(getattr(r, k), getattr(w, k)), k
    M.close()
    # a column of A with more than 512 entries: A^T has a long row, which stays
    # on the long-slice kernel, so the sweep is off
    m, n = 1200, 2000
    rows = []
    for i in range(m):
        L = 600 if i == 7 else int(rng.integers(1, 20))
        c = np.sort(rng.choice(np.arange(1, n), size=L, replace=False))
        if i % 2 == 0:
            c = np.concatenate([[0], c])  # column 0 appears in 600 rows
        rows.append((c, rng.standard_normal(len(c))))
    rp, ci, va = _csr_from_rows(m, n, rows)
    M = eq.ExplicitMatrix.from_csr(m, n, rp, ci, va)
    assert not eq.sweep_active(M)
    r = eq.sgd_equilibrate(M, eq.EquilibrationParams(iterations=6, seed=1))
    w = oracle.c_oracle().sgd_equilibrate(oracle.CsrArrays(m, n, rp, ci, va), iterations=6, seed=1)
    for k in "uvde":
        assert np.array_equal(getattr(r, k), getattr(w, k)), k
    M.close()


def test_sweep_few_long_rows_and_boundaries():
    """Fewer long rows than SMs, run lengths around the unroll, rows of exactly
    513 entries, an empty panel range."""
    rng = np.random.default_rng(4)
    m, n = 500, 6000
    rows = []
    for i in range(m):
        if i in (3, 77, 78, 400):
            L = (513, 514, 2999, 1024)[(3, 77, 78, 400).index(i)]
            # keep the first 1500 columns empty for two of them (empty runs)
            lo = 1500 if i in (77, 400) else 0
            c = np.sort(rng.choice(np.arange(lo, n), size=L, replace=False))
        else:
            L = int(rng.integers(0, 12))
            c = np.sort(rng.choice(n, size=L, replace=False))
        rows.append((c, rng.standard_normal(len(c))))
    rp, ci, va = _csr_from_rows(m, n, rows)
    want = oracle.c_oracle().sgd_equilibrate(oracle.CsrArrays(m, n, rp, ci, va), iterations=8, seed=9)
    for env in ({}, {"EQUIL_SWEEP_WIDTH": "256"}, {"EQUIL_SWEEP_WIDTH": "512", "EQUIL_SWEEP_STAGES": "4"}):
        def go():
            M = eq.ExplicitMatrix.from_csr(m, n, rp, ci, va)
            assert eq.sweep_active(M)
            r = eq.sgd_equilibrate(M, eq.EquilibrationParams(iterations=8, seed=9))
            M.close()
            return r
        got = _with_env(dict(env, EQUIL_SWEEP="1"), go)
        for k in "uvde":
            assert np.array_equal(getattr(got, k), getattr(want, k)), (env, k)


def test_one_shot_call_with_and_without_the_sweep(c3s):
    """The one-shot entry point (from 64 iterations it plans the sweep and leaves A's
    long interleaved slices out): with the sweep, with the sweep layout failing after
    the slices were left out (EQUIL_SWEEP_FAIL: they are completed for the long-slice
    kernel), and under 64 iterations (no sweep) -- all bit-identical to the oracle."""
    inst = c3s
    A = oracle.CsrArrays(inst.m, inst.n, inst.row_ptr, inst.col, inst.val)
    for T, env in ((64, {}), (64, {"EQUIL_SWEEP_FAIL": "1"}), (20, {})):
        want = oracle.c_oracle().sgd_equilibrate(A, iterations=T, seed=8)
        got = _with_env(env, lambda: eq.sgd_equilibrate_csr(
            inst.m, inst.n, inst.row_ptr, inst.col, inst.val,
            eq.EquilibrationParams(iterations=T, seed=8)))
        for k in "uvde":
            assert np.array_equal(getattr(got, k), getattr(want, k)), (T, env, k)


@pytest.mark.parametrize("seed", range(10))
def test_sweep_random_instances_match_long_kernel(seed):
    """Random shapes, long-row counts, panel widths and stage counts: the sweep
    and the long-slice kernel give the same u, v, d, e bit for bit (both are
    pinned to the oracle elsewhere; here the two device paths check each other)."""
    rng = np.random.default_rng(100 + seed)
    m = int(rng.integers(200, 3000))
    n = 2 * int(rng.integers(600, 12000))  # even
    nlong = int(rng.integers(1, 300))
    rows = []
    long_at = set(rng.choice(m, size=min(nlong, m), replace=False).tolist())
    for i in range(m):
        if i in long_at:
            L = int(rng.integers(513, min(n, 6000) + 1))
        else:
            # keep every column short: few entries per ordinary row
            L = int(rng.integers(0, 8))
        c = np.sort(rng.choice(n, size=L, replace=False))
        rows.append((c, rng.standard_normal(L) * np.exp(rng.standard_normal(L))))
    rp, ci, va = _csr_from_rows(m, n, rows)
    # the sweep needs A^T free of long rows: cap the column counts
    counts = np.bincount(ci, minlength=n)
    if counts.max() > 512:
        pytest.skip("instance has a long column")
    width = [None, 128, 192, 300, 1024, 4096][seed % 6]
    env = {"EQUIL_SWEEP": "1", "EQUIL_SWEEP_STAGES": str(2 + seed % 3)}
    if width:
        env["EQUIL_SWEEP_WIDTH"] = str(width)
    p = eq.EquilibrationParams(iterations=7, seed=seed)

    def run(envs, expect_on):
        def go():
            M = eq.ExplicitMatrix.from_csr(m, n, rp, ci, va)
            assert eq.sweep_active(M) == expect_on
            r = eq.sgd_equilibrate(M, p)
            M.close()
            return r
        return _with_env(envs, go)

    got = run(env, True)
    base = run({"EQUIL_SWEEP": "0"}, False)
    for k in "uvde":
        assert np.array_equal(getattr(got, k), getattr(base, k)), (seed, k)
