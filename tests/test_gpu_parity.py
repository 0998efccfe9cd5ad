"""GPU parity: the CUDA path (through the C ABI) against the oracle and the
reference's golden vectors.  Bit-exact for signs, transpose and the whole
SGD / LSQR trajectories (SURVEY.md §0 fact 4 explains why nothing weaker
survives the chaotic recurrence); diagnostics to 1e-12 relative (no feedback,
different summation order and exp)."""
import numpy as np
import pytest

import oracle
import paper_1602_06621_b200 as eq
from conftest import csr_from_golden

pytestmark = pytest.mark.gpu

CASES = ["sp", "lr", "dn"]


def device_matrix(A: oracle.CsrArrays):
    if A.dense is not None:
        return eq.ExplicitMatrix.dense(A.dense)
    return eq.ExplicitMatrix.from_csr(A.m, A.n, A.row_ptr, A.col, A.val)


def bits_of(raw, start, count):
    return np.array([(int(raw[start + k]) >> 63) for k in range(count)], np.uint8)


def unpack(words, count):
    return np.array([(int(words[k >> 5]) >> (k & 31)) & 1 for k in range(count)], np.uint8)


# ---------------------------------------------------------------- K1 signs
def test_sign_stream_matches_reference_outputs(golden):
    raw = golden["raw_0_17"]
    for start, count in [(0, 20000), (1, 31), (312, 5000), (7777, 3333)]:
        got = unpack(eq.sign_bits(0, 17, start, count), count)
        assert np.array_equal(got, bits_of(raw, start, count)), (start, count)
    raw1 = golden["raw_1_17"]
    assert np.array_equal(unpack(eq.sign_bits(1, 17, 0, 20000), 20000), bits_of(raw1, 0, 20000))


@pytest.mark.parametrize("seed,start,count", [(0, 1_000_000 - 5, 4096), (0, 3_000_000, 2048),
                                              (7, 12_345_678, 1000), (99, 0, 2_000_000)])
def test_sign_stream_far_positions_match_oracle(C, seed, start, count):
    """jump-ahead (many segments, several levels) vs sequential generation"""
    got = eq.sign_bits(seed, 17, start, count)
    want = C.sign_bits(seed, 17, start, count)
    assert np.array_equal(got, want)


def test_sign_stream_survey_kats():
    # output [1e6] of (0,17) has MSB 1 (+), [3e8] of (0,17) +, (1,17)[3e8] +
    assert unpack(eq.sign_bits(0, 17, 1_000_000, 1), 1)[0] == 1
    assert unpack(eq.sign_bits(0, 17, 3_000_000, 1), 1)[0] == 0
    assert unpack(eq.sign_bits(0, 17, 10_000_000, 1), 1)[0] == 0


# ---------------------------------------------------------------- K2 transpose
@pytest.mark.parametrize("key", ["sp", "lr"])
def test_transpose_bit_exact_vs_reference(golden, key):
    A = csr_from_golden(golden, key)
    M = device_matrix(A)
    trp, tc, tv = M.transposed_csr()
    assert np.array_equal(trp, golden[f"{key}_t_rp"])
    assert np.array_equal(tc, golden[f"{key}_t_col"])
    assert np.array_equal(tv.view(np.uint64), golden[f"{key}_t_val"].view(np.uint64))


def test_transpose_bit_exact_config1(C):
    from paper_1602_06621_b200 import configs
    inst = configs.config(1)
    A = oracle.CsrArrays(inst.m, inst.n, inst.row_ptr, inst.col, inst.val)
    T = C.transpose(A)
    trp, tc, tv = device_matrix(A).transposed_csr()
    assert np.array_equal(trp, T.row_ptr) and np.array_equal(tc, T.col)
    assert np.array_equal(tv.view(np.uint64), T.val.view(np.uint64))


# ---------------------------------------------------------------- numerics contract
def test_det_exp_device_equals_oracle(C):
    rng = np.random.default_rng(3)
    x = np.concatenate([rng.uniform(-20, 20, 200_000), rng.standard_normal(50_000) * 1e-3,
                        np.array([0.0, -0.0, 9.210340371976184, -9.210340371976184, 709.0,
                                  -707.0, 1e-300, -1e-300])])
    got = eq.det_exp_device(x)
    want = C.det_exp(x)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


@pytest.mark.parametrize("n", [0, 1, 255, 2048, 2049, 100_000, 2048 * 1024 + 17])
def test_canonical_reduction_device_equals_oracle(C, n):
    x = np.random.default_rng(n).standard_normal(n) * 3.0
    assert eq.canon_sumsq_device(x) == C.canon_sumsq(x)


# ---------------------------------------------------------------- apply / adjoint
@pytest.mark.parametrize("key", CASES)
def test_apply_and_adjoint_bit_exact(C, golden, key):
    A = csr_from_golden(golden, key)
    M = device_matrix(A)
    rng = np.random.default_rng(1)
    x = rng.standard_normal(A.n)
    y = rng.standard_normal(A.m)
    assert np.array_equal(M.apply(x), C.apply(A, x))
    assert np.array_equal(M.apply_adjoint(y), C.apply(A, y, adjoint=True))


# ---------------------------------------------------------------- SGD trajectory
@pytest.mark.parametrize("key", CASES)
def test_sgd_bit_exact_vs_reference_golden(golden, key):
    A = csr_from_golden(golden, key)
    M = device_matrix(A)
    r = eq.sgd_equilibrate(M, eq.EquilibrationParams(iterations=40, seed=5))
    for k in "uvde":
        assert np.array_equal(getattr(r, k), golden[f"{key}_sgd_{k}"]), k
    box, bound, ap, ad = golden[f"{key}_sgd_flags"]
    assert (r.box_feasible, r.iterate_bound_ok, r.apply_count, r.adjoint_count) == \
        (bool(box), bool(bound), ap, ad)


def test_sgd_history_within_tolerance(golden):
    A = csr_from_golden(golden, "sp")
    M = device_matrix(A)
    r = eq.sgd_equilibrate(M, eq.EquilibrationParams(iterations=40, seed=5),
                           eq.DiagnosticsConfig(stride=10))
    assert [h.iter for h in r.history] == [0, 10, 20, 30, 40]
    rms = np.array([h.rms for h in r.history])
    obj = np.array([h.objective for h in r.history])
    np.testing.assert_allclose(rms, golden["sp_sgd_hist_rms"], rtol=1e-12, atol=0)
    np.testing.assert_allclose(obj, golden["sp_sgd_hist_obj"], rtol=1e-12, atol=0)
    for k in "uvde":  # history must not perturb the trajectory
        assert np.array_equal(getattr(r, k), golden[f"sp_sgd_{k}"])


def test_sgd_config1_bit_exact_vs_oracle(C):
    """BASELINE config 1 (10000x5000, 1%, T=50, seed 0, beta=1, alpha=sqrt(n/m))."""
    from paper_1602_06621_b200 import configs
    inst = configs.config(1)
    A = oracle.CsrArrays(inst.m, inst.n, inst.row_ptr, inst.col, inst.val)
    want = C.sgd_equilibrate(A, alpha=inst.alpha, beta=inst.beta, iterations=50, seed=0)
    M = device_matrix(A)
    p = eq.EquilibrationParams(alpha=inst.alpha, beta=inst.beta, iterations=50, seed=0)
    got = eq.sgd_equilibrate(M, p)
    for k in "uvde":
        assert np.array_equal(getattr(got, k), getattr(want, k)), k
    # graph replay on the same handle is bit-identical (determinism, :229-245)
    again = eq.sgd_equilibrate(M, p)
    assert np.array_equal(again.d, got.d) and np.array_equal(again.e, got.e)
    other = eq.sgd_equilibrate(M, eq.EquilibrationParams(alpha=inst.alpha, beta=inst.beta,
                                                          iterations=50, seed=1))
    assert not np.array_equal(other.u, got.u)


def test_sgd_identity_fixed_point():
    """test_equilibrate.cpp:183-198"""
    M = eq.ExplicitMatrix.identity(5)
    r = eq.sgd_equilibrate(M, eq.EquilibrationParams(alpha=1.0, beta=1.0, iterations=50),
                           eq.DiagnosticsConfig(stride=1))
    assert np.all(r.u == 0) and np.all(r.v == 0) and np.all(r.d == 1) and np.all(r.e == 1)
    assert all(abs(h.objective - 2.5) <= 2.5e-15 for h in r.history)
    assert all(abs(h.rms) <= 1e-15 for h in r.history)


def test_sgd_scalar_and_zero_known_answers(C):
    """test_equilibrate.cpp:200-227 (1x1 [2]) and :302-331 (zero matrix)"""
    one = oracle.CsrArrays(1, 1, dense=np.array([[2.0]]))
    p = eq.EquilibrationParams(alpha=1.0, beta=1.0, gamma=0.1, max_log_scale=10.0,
                               iterations=10000)
    r = eq.sgd_equilibrate(eq.ExplicitMatrix.dense(one.dense), p)
    w = C.sgd_equilibrate(one, alpha=1.0, beta=1.0, gamma=0.1, max_log_scale=10.0,
                          iterations=10000)
    assert np.array_equal(r.u, w.u) and np.array_equal(r.v, w.v)
    assert r.box_feasible and r.iterate_bound_ok
    z = eq.ExplicitMatrix.from_csr(1, 1, np.array([0, 1]), np.array([0]), np.array([0.0]))
    r = eq.sgd_equilibrate(z, eq.EquilibrationParams(alpha=1.0, beta=1.0, iterations=57))
    w = C.sgd_equilibrate(oracle.CsrArrays(1, 1, np.array([0, 1]), np.array([0]),
                                           np.array([0.0])), alpha=1.0, beta=1.0,
                          iterations=57)
    assert np.array_equal(r.u, w.u)


@pytest.mark.parametrize("T", [0, 1, 2])
def test_sgd_tiny_budgets(C, golden, T):
    A = csr_from_golden(golden, "sp")
    r = eq.sgd_equilibrate(device_matrix(A), eq.EquilibrationParams(iterations=T, seed=2))
    w = C.sgd_equilibrate(A, iterations=T, seed=2)
    for k in "uvde":
        assert np.array_equal(getattr(r, k), getattr(w, k))
    assert r.apply_count == T and r.adjoint_count == T


def test_sgd_random_shapes_vs_oracle(C):
    rng = np.random.default_rng(21)
    for m, n, dens in [(1, 7, 0.9), (7, 1, 0.9), (513, 257, 0.02), (2, 3000, 0.8)]:
        mask = rng.random((m, n)) < dens
        a = rng.standard_normal((m, n)) * np.exp(2 * rng.standard_normal((m, 1)))
        rp = np.concatenate([[0], np.cumsum(mask.sum(1))])
        A = oracle.CsrArrays(m, n, rp, np.nonzero(mask)[1], a[mask])
        p = dict(iterations=33, seed=int(rng.integers(1 << 30)))
        w = C.sgd_equilibrate(A, **p)
        r = eq.sgd_equilibrate(device_matrix(A), eq.EquilibrationParams(**p))
        for k in "uvde":
            assert np.array_equal(getattr(r, k), getattr(w, k)), (m, n, k)
        Ad = oracle.CsrArrays(m, n, dense=np.where(mask, a, 0.0))
        w = C.sgd_equilibrate(Ad, **p)
        r = eq.sgd_equilibrate(device_matrix(Ad), eq.EquilibrationParams(**p))
        for k in "uvde":
            assert np.array_equal(getattr(r, k), getattr(w, k)), ("dense", m, n, k)


# ---------------------------------------------------------------- LSQR
@pytest.mark.parametrize("key", CASES)
def test_lsqr_bit_exact_vs_reference_golden(golden, key):
    A = csr_from_golden(golden, key)
    M = device_matrix(A)
    b = golden[f"{key}_b"]
    run = eq.lsqr(M, b, 30, 0.0)
    assert np.array_equal(np.array(run.residual_history), golden[f"{key}_lsqr_res"])
    assert np.array_equal(run.x, golden[f"{key}_lsqr_x"])
    assert [run.iterations, run.reached_tol, run.breakdown, run.apply_count,
            run.adjoint_count] == list(golden[f"{key}_lsqr_meta"])
    pre = eq.lsqr_preconditioned(M, b, eq.EquilibrationParams(iterations=15, seed=3), 30, 0.0)
    assert np.array_equal(np.array(pre.residual_history), golden[f"{key}_plsqr_res"])
    assert np.array_equal(pre.x, golden[f"{key}_plsqr_x"])
    assert [pre.iterations, pre.reached_tol, pre.breakdown, pre.apply_count,
            pre.adjoint_count] == list(golden[f"{key}_plsqr_meta"])


def test_lsqr_reference_cases():
    """test_itersolvers.cpp:36-56, :88-121, :123-142"""
    rng = np.random.default_rng(81)
    b = rng.standard_normal(6)
    run = eq.lsqr(eq.ExplicitMatrix.identity(6), b, 10, 1e-12)
    assert run.reached_tol and run.iterations == 1 and len(run.residual_history) == 2
    assert run.residual_history[0] == 1.0 and run.residual_history[1] <= 1e-12
    assert np.linalg.norm(run.x - b) <= 1e-12 * np.linalg.norm(b)
    D = np.diag(np.arange(1.0, 6.0))
    run = eq.lsqr(eq.ExplicitMatrix.dense(D), D @ np.ones(5), 10, 1e-13)
    assert run.reached_tol and run.iterations <= 5
    assert np.abs(run.x - 1).max() <= 1e-10
    with pytest.raises(eq.InvalidArgument):
        eq.lsqr(eq.ExplicitMatrix.identity(3), np.zeros(3), 5, 1e-6)
    A = np.zeros((2, 2)); A[0, 0] = 1.0
    run = eq.lsqr(eq.ExplicitMatrix.dense(A), np.array([0.0, 1.0]), 20, 1e-10)
    assert run.breakdown and not run.reached_tol and run.iterations == 0
    assert np.linalg.norm(run.x) == 0 and run.residual_history == [1.0]
    run = eq.lsqr(eq.ExplicitMatrix.dense(A), np.array([1.0, 1.0]), 20, 1e-10)
    assert not run.reached_tol and abs(run.x[0] - 1) < 1e-12 and abs(run.x[1]) < 1e-12
    assert run.residual_history[-1] == pytest.approx(1 / np.sqrt(2), rel=1e-12)
    b = np.random.default_rng(84).standard_normal(7)
    I7 = eq.ExplicitMatrix.identity(7)
    plain = eq.lsqr(I7, b, 50, 1e-12)
    pre = eq.lsqr_preconditioned(I7, b, eq.EquilibrationParams(iterations=9), 50, 1e-12)
    assert pre.equil_iterations == 9 and np.array_equal(pre.x, plain.x)
    assert pre.residual_history[:10] == [1.0] * 10
    assert pre.residual_history[10:] == plain.residual_history[1:]
    assert pre.apply_count == plain.apply_count + 9
    assert pre.adjoint_count == plain.adjoint_count + 9


# ---------------------------------------------------------------- errors
def test_errors_mirror_reference():
    with pytest.raises(eq.InvalidArgument, match="duplicate"):
        eq.ExplicitMatrix.from_csr(2, 2, [0, 2, 2], [1, 1], [1.0, 2.0])
    with pytest.raises(eq.InvalidArgument, match="out of range"):
        eq.ExplicitMatrix.from_csr(2, 2, [0, 1, 1], [5], [1.0])
    with pytest.raises(eq.InvalidArgument, match="duplicate"):
        eq.ExplicitMatrix.sparse(2, 2, [(0, 1, 1.0), (0, 1, 2.0)])
    M = eq.ExplicitMatrix.identity(3)
    with pytest.raises(eq.InvalidArgument, match="gamma"):
        eq.sgd_equilibrate(M, eq.EquilibrationParams(gamma=-1.0, iterations=1))
    with pytest.raises(eq.InvalidArgument, match="violated"):
        eq.sgd_equilibrate(M, eq.EquilibrationParams(alpha=1.0, beta=2.0, iterations=1))
    with pytest.raises(eq.InvalidArgument, match="nonnegative"):
        eq.sgd_equilibrate(M, eq.EquilibrationParams(iterations=-1))


# ---------------------------------------------------------------- larger scales
def test_sgd_scaled_config3_bit_exact(C):
    """c3's generator at 2% scale (40000 x 20000, Zipf rows up to 1e4: long-row
    CTA slices, slices, empty columns) -- full trajectory bit-exact."""
    from paper_1602_06621_b200 import configs
    inst = configs.config(3, scale=0.02)
    A = oracle.CsrArrays(inst.m, inst.n, inst.row_ptr, inst.col, inst.val)
    assert np.diff(inst.row_ptr).max() > 2048
    want = C.sgd_equilibrate(A, iterations=20, seed=7)
    got = eq.sgd_equilibrate(device_matrix(A), eq.EquilibrationParams(iterations=20, seed=7))
    for k in "uvde":
        assert np.array_equal(getattr(got, k), getattr(want, k)), k
    assert (got.box_feasible, got.iterate_bound_ok) == (want.box_feasible, want.iterate_bound_ok)


@pytest.mark.parametrize("case", ["sp", "lr", "c3"])
@pytest.mark.parametrize("lvariant", ["2", "3"])
def test_long_slice_variants_bit_exact(C, golden, monkeypatch, case, lvariant):
    """The long-slice ring at other shapes than the default (EQUIL_SELL_LVARIANT:
    2 entries x 15 stagers, 4 x 7 with four CTAs per SM): same trajectory bit for
    bit -- golden cases and c3's generator at 2% scale (rows of up to 10^4
    entries), so the ring protocol does not depend on its shape."""
    monkeypatch.setenv("EQUIL_SELL_LVARIANT", lvariant)
    monkeypatch.setenv("EQUIL_SWEEP", "0")  # the SGD's long rows on the long-slice kernel
    if case == "c3":
        from paper_1602_06621_b200 import configs
        inst = configs.config(3, scale=0.02)
        A = oracle.CsrArrays(inst.m, inst.n, inst.row_ptr, inst.col, inst.val)
        want = C.sgd_equilibrate(A, iterations=20, seed=7)
        got = eq.sgd_equilibrate(device_matrix(A), eq.EquilibrationParams(iterations=20, seed=7))
        want = {k: getattr(want, k) for k in "uvde"}
    else:
        A = csr_from_golden(golden, case)
        got = eq.sgd_equilibrate(device_matrix(A), eq.EquilibrationParams(iterations=40, seed=5))
        want = {k: golden[f"{case}_sgd_{k}"] for k in "uvde"}
    for k in "uvde":
        assert np.array_equal(getattr(got, k), want[k]), k


def test_lsqr_config1_bit_exact(C):
    from paper_1602_06621_b200 import configs
    inst = configs.config(1)
    A = oracle.CsrArrays(inst.m, inst.n, inst.row_ptr, inst.col, inst.val)
    b = configs.rhs(inst)
    M = device_matrix(A)
    run = eq.lsqr(M, b, 25, 0.0)
    ref = C.lsqr(A, b, 25, 0.0)
    assert np.array_equal(np.array(run.residual_history), ref.residual_history)
    assert np.array_equal(run.x, ref.x)
    pre = eq.lsqr_preconditioned(M, b, eq.EquilibrationParams(iterations=10, seed=2), 25, 0.0)
    pref = C.lsqr_preconditioned(A, b, 25, 0.0, iterations=10, seed=2)
    assert np.array_equal(np.array(pre.residual_history), pref.residual_history)
    assert np.array_equal(pre.x, pref.x)
    assert (pre.apply_count, pre.adjoint_count) == (pref.apply_count, pref.adjoint_count)


def test_full_size_config3_properties(C):
    """BASELINE size (2e6 x 1e6, nnz 1.5e8): size-independent properties --
    bit-for-bit determinism across handles and entry points, d = det_exp(u)
    exactly, the box, and the reference's flags."""
    from paper_1602_06621_b200 import configs
    inst = configs.config(3)
    p = eq.EquilibrationParams(iterations=5, seed=0)
    M = eq.ExplicitMatrix.from_csr(inst.m, inst.n, inst.row_ptr, inst.col, inst.val)
    r1 = eq.sgd_equilibrate(M, p)
    r2 = eq.sgd_equilibrate(M, p)
    r3 = eq.sgd_equilibrate_csr(inst.m, inst.n, inst.row_ptr, inst.col, inst.val, p)
    for k in "uvde":
        assert np.array_equal(getattr(r1, k), getattr(r2, k))
        assert np.array_equal(getattr(r1, k), getattr(r3, k))
    idx = np.random.default_rng(0).integers(0, inst.m, 20000)
    assert np.array_equal(r1.d[idx], C.det_exp(r1.u[idx]))
    assert np.abs(r1.u).max() <= p.max_log_scale and np.abs(r1.v).max() <= p.max_log_scale
    assert r1.box_feasible and r1.iterate_bound_ok
    # the transpose of the full matrix is a permutation of A's entries by column
    trp, tc, tv = M.transposed_csr()
    assert trp[-1] == inst.nnz and np.all(np.diff(trp) >= 0)
    assert np.array_equal(np.diff(trp), np.bincount(inst.col, minlength=inst.n))


# ---------------------------------------------------------------- targets variant (f4)
def test_targets_variant_bit_exact_vs_reference_golden(golden):
    A = csr_from_golden(golden, "sp")
    M = device_matrix(A)
    r = eq.sgd_equilibrate_targets(M, golden["tg_r"], golden["tg_c"],
                                   eq.EquilibrationParams(iterations=30, seed=4),
                                   eq.DiagnosticsConfig(stride=10))
    for k in "uvde":
        assert np.array_equal(getattr(r, k), golden[f"tg_sgd_{k}"]), k
    np.testing.assert_allclose([h.objective for h in r.history], golden["tg_sgd_hist_obj"],
                               rtol=1e-12)
    assert all(h.rms is None for h in r.history) and (r.alpha, r.beta) == (0.0, 0.0)
    box, bound, ap, ad = golden["tg_sgd_flags"]
    assert (r.box_feasible, r.iterate_bound_ok, r.apply_count) == (bool(box), bool(bound), ap)
    # without history the graph path gives the same trajectory
    r2 = eq.sgd_equilibrate_targets(M, golden["tg_r"], golden["tg_c"],
                                    eq.EquilibrationParams(iterations=30, seed=4))
    assert np.array_equal(r2.u, r.u) and np.array_equal(r2.e, r.e)
    # and the uniform path on the same handle is unaffected afterwards
    u = eq.sgd_equilibrate(M, eq.EquilibrationParams(iterations=40, seed=5))
    assert np.array_equal(u.u, golden["sp_sgd_u"])
    with pytest.raises(eq.InvalidArgument, match="sum"):
        eq.sgd_equilibrate_targets(M, golden["tg_r"], 2 * golden["tg_c"])
    with pytest.raises(eq.InvalidArgument, match="positive"):
        eq.sgd_equilibrate_targets(M, -golden["tg_r"], golden["tg_c"])


def test_targets_variant_dense_vs_oracle(C, golden):
    A = csr_from_golden(golden, "dn")
    rng = np.random.default_rng(8)
    rr = rng.uniform(0.2, 3.0, A.m)
    cc = rng.uniform(0.2, 3.0, A.n)
    cc *= rr.sum() / cc.sum()
    want = C.sgd_equilibrate_targets(A, rr, cc, iterations=25, seed=9)
    got = eq.sgd_equilibrate_targets(device_matrix(A), rr, cc,
                                     eq.EquilibrationParams(iterations=25, seed=9))
    for k in "uvde":
        assert np.array_equal(getattr(got, k), getattr(want, k)), k


# ---------------------------------------------------------------- COO ingest (f2)
def test_coo_ingest_equals_reference_construction(golden):
    """ExplicitMatrix::sparse from shuffled COO triplets on device: same CSR
    (hence same CSR(A^T) and trajectory) as the reference's construction."""
    A = csr_from_golden(golden, "lr")
    rows = np.repeat(np.arange(A.m), np.diff(A.row_ptr))
    perm = np.random.default_rng(5).permutation(rows.size)
    M = eq.ExplicitMatrix.sparse(A.m, A.n, (rows[perm], A.col[perm].astype(np.int64),
                                            A.val[perm]))
    trp, tc, tv = M.transposed_csr()
    assert np.array_equal(trp, golden["lr_t_rp"]) and np.array_equal(tc, golden["lr_t_col"])
    assert np.array_equal(tv.view(np.uint64), golden["lr_t_val"].view(np.uint64))
    r = eq.sgd_equilibrate(M, eq.EquilibrationParams(iterations=40, seed=5))
    for k in "uvde":
        assert np.array_equal(getattr(r, k), golden[f"lr_sgd_{k}"])


def test_coo_errors_match_reference_messages():
    cases = [
        (3, 3, [(0, 0, 1.0), (5, 1, 1.0), (3, 3, 2.0)]),          # first bad in input order
        (3, 3, [(2, 2, 1.0), (0, 1, 2.0), (2, 2, 3.0), (0, 1, 4.0)]),  # first dup after sort
        (2, 4, [(1, -1, 1.0)]),
    ]
    want = ["ExplicitMatrix::sparse: entry (5, 1) out of range",
            "ExplicitMatrix::sparse: duplicate entry (0, 1)",
            "ExplicitMatrix::sparse: entry (1, -1) out of range"]
    for (m, n, ent), msg in zip(cases, want):
        with pytest.raises(eq.InvalidArgument) as ei:
            eq.ExplicitMatrix.sparse(m, n, ent)
        assert str(ei.value) == msg
        if oracle.ref_available():  # the reference's own construction agrees
            r, c, v = (np.array(x) for x in zip(*ent))
            with pytest.raises(oracle.OracleError) as er:
                oracle.ref_oracle().matrix_coo(m, n, r, c, v)
            assert str(er.value) == msg
    # empty rows/columns and an empty matrix are fine
    M = eq.ExplicitMatrix.sparse(4, 3, [])
    assert M.stored_entries() == 0
    r = eq.sgd_equilibrate(M, eq.EquilibrationParams(alpha=1.0, iterations=3))
    assert np.all(r.u < 0) or np.all(r.u != 0)


# ---------------------------------------------------------------- engine variants
def test_symmetric_variant_bit_exact_vs_reference_golden(golden):
    """sgd_equilibrate_symmetric (src/variants.cpp:35-103) on the device."""
    S = csr_from_golden(golden, "sy")
    r = eq.sgd_equilibrate_symmetric(device_matrix(S), eq.EquilibrationParams(iterations=40,
                                                                              seed=6),
                                     eq.DiagnosticsConfig(stride=10))
    for k in "uvde":
        assert np.array_equal(getattr(r, k), golden[f"sy_sgd_{k}"]), k
    box, bound, ap, ad = golden["sy_sgd_flags"]
    assert (r.box_feasible, r.iterate_bound_ok, r.apply_count, r.adjoint_count) == \
        (bool(box), bool(bound), ap, ad)
    np.testing.assert_allclose([h.objective for h in r.history], golden["sy_sgd_hist_obj"],
                               rtol=1e-12, atol=0)
    np.testing.assert_allclose([h.rms for h in r.history], golden["sy_sgd_hist_rms"],
                               rtol=1e-12, atol=0)


def test_block_variant_bit_exact_vs_reference_golden(golden):
    """sgd_equilibrate_block (src/variants.cpp:156-240) on the device."""
    A = csr_from_golden(golden, "sp")
    rb, cb = golden["bl_rb"], golden["bl_cb"]
    st = eq.BlockStructure(rb, cb, 17, int(cb.max()) + 1)
    r = eq.sgd_equilibrate_block(device_matrix(A), st, eq.EquilibrationParams(iterations=30,
                                                                              seed=8),
                                 eq.DiagnosticsConfig(stride=10))
    for k in "uvde":
        assert np.array_equal(getattr(r, k), golden[f"bl_sgd_{k}"]), k
    np.testing.assert_allclose([h.objective for h in r.history], golden["bl_sgd_hist_obj"],
                               rtol=1e-12, atol=0)
    np.testing.assert_allclose([h.rms for h in r.history], golden["bl_sgd_hist_rms"],
                               rtol=1e-12, atol=0)


def test_variants_dense_and_known_answers_vs_oracle(C):
    """Dense operands, singleton blocks == the plain solver, identity fixed
    point, and the reference's rejections (test_variants.cpp:36-61, :165-176,
    :234-249)."""
    rng = np.random.default_rng(5)
    X = rng.standard_normal((48, 48)) * np.exp(rng.standard_normal((48, 1)))
    Sd = np.triu(X) + np.triu(X, 1).T
    A = oracle.CsrArrays(48, 48, dense=Sd)
    want = C.sgd_equilibrate_symmetric(A, iterations=60, seed=2)
    got = eq.sgd_equilibrate_symmetric(eq.ExplicitMatrix.dense(Sd),
                                       eq.EquilibrationParams(iterations=60, seed=2))
    for k in "uvde":
        assert np.array_equal(getattr(got, k), getattr(want, k)), k
    D = rng.standard_normal((40, 25)) * np.exp(2 * rng.standard_normal((40, 1)))
    B = oracle.CsrArrays(40, 25, dense=D)
    rb, cb = np.arange(40) % 6, np.arange(25) // 5
    want = C.sgd_equilibrate_block(B, rb, cb, 6, 5, iterations=50, seed=3)
    got = eq.sgd_equilibrate_block(eq.ExplicitMatrix.dense(D), eq.BlockStructure(rb, cb, 6, 5),
                                   eq.EquilibrationParams(iterations=50, seed=3))
    for k in "uvde":
        assert np.array_equal(getattr(got, k), getattr(want, k)), k
    M = eq.ExplicitMatrix.dense(D)
    plain = eq.sgd_equilibrate(M, eq.EquilibrationParams(iterations=40, seed=11))
    blk = eq.sgd_equilibrate_block(M, eq.BlockStructure.trivial(40, 25),
                                   eq.EquilibrationParams(iterations=40, seed=11))
    for k in "uvde":
        assert np.array_equal(getattr(plain, k), getattr(blk, k)), k
    r = eq.sgd_equilibrate_symmetric(eq.ExplicitMatrix.identity(4),
                                     eq.EquilibrationParams(alpha=1.0, beta=1.0,
                                                            iterations=100))
    assert np.all(r.u == 0) and np.array_equal(r.d, r.e) and (r.apply_count,
                                                               r.adjoint_count) == (100, 0)
    with pytest.raises(eq.InvalidArgument, match="symmetry check"):
        eq.sgd_equilibrate_symmetric(eq.ExplicitMatrix.dense(rng.standard_normal((5, 5))),
                                     eq.EquilibrationParams(alpha=1.0, beta=1.0))
    with pytest.raises(eq.InvalidArgument, match="must be square"):
        eq.sgd_equilibrate_symmetric(eq.ExplicitMatrix.dense(np.ones((3, 4))),
                                     eq.EquilibrationParams(alpha=1.0, beta=1.0))
    Bm = eq.ExplicitMatrix.dense(rng.standard_normal((3, 2)) + 1.5)
    for rbx, cbx, R, Cb, msg in [([0, 0, 1], [0, 1], 3, 2, "empty row block"),
                                 ([0, 0, 1], [0, 1], 1, 2, "row block index out of range"),
                                 ([0, 0, 1], [0, -1], 2, 2, "col block index out of range"),
                                 ([0, 0, 1, 1], [0, 1], 2, 2, "assignment length mismatch")]:
        with pytest.raises(eq.InvalidArgument, match=msg):
            eq.sgd_equilibrate_block(Bm, eq.BlockStructure(np.array(rbx), np.array(cbx), R, Cb),
                                     eq.EquilibrationParams(iterations=3))


# ---------------------------------------------------------------- CCP lasso
@pytest.mark.parametrize("key", ["sp", "dn"])
def test_ccp_and_spectral_norm_bit_exact_vs_reference_golden(golden, key):
    """spectral_norm (src/lsqr.cpp:140-163), ccp_lasso and
    ccp_lasso_preconditioned (src/ccp.cpp:27-141) on the device: plain,
    preconditioned and gap-stopped runs, every history entry bit-exact."""
    A = csr_from_golden(golden, key)
    M = device_matrix(A)
    b = golden[f"{key}_b"]
    sn = golden[f"{key}_snorm"]
    assert eq.spectral_norm(M, 100, 1e-9, 0) == sn[0]
    assert eq.spectral_norm(M, 300, 1e-12, 1) == sn[1]
    ps = float(golden[f"{key}_pstar"][0])
    prob = eq.LassoProblem(M, b, 0.3)
    for tag, opt, params in [
            ("ccp", eq.CcpOptions(max_iters=150, p_star=ps), None),
            ("pccp", eq.CcpOptions(max_iters=150, p_star=ps),
             eq.EquilibrationParams(iterations=30, seed=3)),
            ("eccp", eq.CcpOptions(max_iters=20000, p_star=ps, gap_tol=1e-4), None)]:
        r = eq.ccp_lasso(prob, opt) if params is None else eq.ccp_lasso_preconditioned(
            prob, params, opt)
        assert np.array_equal(r.x, golden[f"{key}_{tag}_x"]), tag
        assert np.array_equal(r.objective_history, golden[f"{key}_{tag}_obj"]), tag
        assert np.array_equal(r.gap_history, golden[f"{key}_{tag}_gap"]), tag
        assert [r.iterations, r.equil_iterations, r.reached_tol, r.apply_count,
                r.adjoint_count] == list(golden[f"{key}_{tag}_meta"]), tag
        assert [r.tau, r.sigma, r.theta] == list(golden[f"{key}_{tag}_steps"]), tag


def test_ccp_known_answers_and_errors(C):
    """test_itersolvers.cpp:173-227, :273-292 on the device."""
    assert eq.spectral_norm(eq.ExplicitMatrix.dense(np.diag([3.0, 1.0])), 500,
                            1e-12) == pytest.approx(3.0, rel=1e-8)
    eye = eq.ExplicitMatrix.identity(2)
    prob = eq.LassoProblem(eye, np.array([3.0, 0.0]), 4.0)
    assert eq.lasso_objective(prob, np.zeros(2)) == pytest.approx(4.5, rel=1e-14)
    assert eq.lasso_objective(prob, np.array([1.0, 0.0])) == pytest.approx(4.0, rel=1e-14)
    r = eq.ccp_lasso(prob, eq.CcpOptions(max_iters=5000))
    assert r.x[0] == pytest.approx(1.0, rel=1e-6) and abs(r.x[1]) <= 1e-8
    assert len(r.objective_history) == r.iterations + 1 and r.gap_history == []
    assert r.apply_count == r.adjoint_count == r.iterations
    rng = np.random.default_rng(91)
    Ad = rng.standard_normal((10, 14))
    bb = rng.standard_normal(10)
    M = eq.ExplicitMatrix.dense(Ad)
    p2 = eq.LassoProblem(M, bb, 0.05)
    plain = eq.ccp_lasso(p2, eq.CcpOptions(max_iters=500))
    pre = eq.ccp_lasso_preconditioned(p2, eq.EquilibrationParams(iterations=0),
                                      eq.CcpOptions(max_iters=500))
    want = C.ccp_lasso(oracle.CsrArrays(10, 14, dense=Ad), bb, 0.05, max_iters=500)
    assert np.array_equal(plain.x, want.x) and np.array_equal(plain.objective_history,
                                                                want.objective_history)
    assert pre.equil_iterations == 0 and np.array_equal(pre.x, plain.x)
    x = rng.standard_normal(14)
    assert eq.lasso_objective(p2, x) == C.lasso_objective(oracle.CsrArrays(10, 14, dense=Ad),
                                                          bb, 0.05, x)
    with pytest.raises(eq.InvalidArgument, match="lambda must be positive"):
        eq.ccp_lasso(eq.LassoProblem(M, bb, 0.0))
    with pytest.raises(eq.InvalidArgument, match="rhs must be nonzero"):
        eq.ccp_lasso(eq.LassoProblem(M, np.zeros(10), 0.1))
    with pytest.raises(eq.InvalidArgument, match="max_iters must be nonnegative"):
        eq.ccp_lasso(p2, eq.CcpOptions(max_iters=-1))
    with pytest.raises(eq.InvalidArgument, match="max_iters must be positive"):
        eq.spectral_norm(M, 0)


# ---------------------------------------------------------------- matrix store
def test_matrix_market_and_binary_ingest_on_device(C, golden, tmp_path):
    """read_matrix_market_file (src/matrix_market.cpp:63-204) through the
    device COO ingest: same matrix as the reference construction (CSR and
    CSR(A^T)), duplicates reported at the later line (:142-158), writer bytes
    equal to what the host writer produces, binary CSR round trip."""
    A = csr_from_golden(golden, "lr")
    rows = np.repeat(np.arange(A.m), np.diff(A.row_ptr))
    perm = np.random.default_rng(0).permutation(A.nnz)  # any entry order
    lines = ["%%MatrixMarket matrix coordinate real general\n", "% shuffled\n",
             f"{A.m} {A.n} {A.nnz}\n"]
    lines += [f"{rows[k] + 1} {A.col[k] + 1} {float(A.val[k])!r}\n" for k in perm]
    p = tmp_path / "lr.mtx"
    p.write_text("".join(lines))
    M = eq.ExplicitMatrix.read_matrix_market(str(p))
    rp, ci, va = M.to_csr()
    assert np.array_equal(rp, A.row_ptr) and np.array_equal(ci, A.col)
    assert np.array_equal(va, A.val)
    trp, tci, tva = M.transposed_csr()
    assert np.array_equal(trp, golden["lr_t_rp"]) and np.array_equal(tva, golden["lr_t_val"])
    r = eq.sgd_equilibrate(M, eq.EquilibrationParams(iterations=40, seed=5))
    assert np.array_equal(r.u, golden["lr_sgd_u"])
    # writer from the device copy == host writer == reference bytes (CPU test)
    w1, w2 = tmp_path / "w1.mtx", tmp_path / "w2.mtx"
    M.write_matrix_market(str(w1))
    eq.write_matrix_market_csr(str(w2), A.m, A.n, A.row_ptr, A.col, A.val)
    assert w1.read_bytes() == w2.read_bytes()
    # binary CSR round trip
    b = tmp_path / "lr.eqb"
    M.save_binary(str(b))
    M2 = eq.ExplicitMatrix.load_binary(str(b))
    assert all(np.array_equal(x, y) for x, y in zip(M2.to_csr(), (A.row_ptr, A.col, A.val)))
    D = golden["dn_dense"]
    Md = eq.ExplicitMatrix.dense(D)
    Md.save_binary(str(b))
    assert np.array_equal(eq.ExplicitMatrix.load_binary(str(b)).to_dense(), D)
    Md.write_matrix_market(str(w1))
    assert np.array_equal(eq.ExplicitMatrix.read_matrix_market(str(w1)).to_dense(), D)
    # duplicates: the first duplicated (row, col) in sorted order, at its later line
    dup = ["%%MatrixMarket matrix coordinate real general\n", "3 3 5\n", "3 3 1.0\n",
           "1 2 1.0\n", "2 2 1.0\n", "% c\n", "1 2 5.0\n", "3 3 2.0\n"]
    p.write_text("".join(dup))
    with pytest.raises(eq.EquilRuntimeError, match=r"line 7: duplicate entry \(1, 2\)"):
        eq.ExplicitMatrix.read_matrix_market(str(p))


# ---------------------------------------------------------------- public helpers
@pytest.mark.parametrize("key", ["sp", "dn"])
def test_equilibrate_helpers_vs_reference_golden(golden, key):
    """stochastic_gradient_estimate (src/equilibrate.cpp:60-71) bit-exact on the
    device; objective / gradient (:10-57) and rms_error (metrics.cpp:41-56) to
    1e-12 relative (the reference uses std::exp and plain sequential sums)."""
    A = csr_from_golden(golden, key)
    M = device_matrix(A)
    u, v = golden[f"{key}_hu"], golden[f"{key}_hv"]
    rng = eq.SeededRng(7, 17)
    rng.position = 123
    su, sv = eq.stochastic_gradient_estimate(M, u, v, eq.EquilibrationParams(), rng)
    assert np.array_equal(su, golden[f"{key}_hsu"]) and np.array_equal(sv, golden[f"{key}_hsv"])
    assert rng.position == 123 + A.m + A.n
    if A.dense is not None:
        with pytest.raises(eq.InvalidArgument, match="sparse matrices only"):
            eq.objective(M, u, v)
        return
    obj = eq.objective(M, u, v)
    assert obj == pytest.approx(golden[f"{key}_hobj"][0], rel=1e-12)
    obj2 = eq.objective(M, u, v, eq.EquilibrationParams(alpha=0.9, gamma=0.3))
    assert obj2 == pytest.approx(golden[f"{key}_hobj"][1], rel=1e-12)
    gu, gv = eq.gradient(M, u, v)
    np.testing.assert_allclose(gu, golden[f"{key}_hgu"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(gv, golden[f"{key}_hgv"], rtol=1e-12, atol=1e-12)
    assert eq.rms_error(M, u, v, 0.7, 1.1) == pytest.approx(golden[f"{key}_hrms"][0], rel=1e-12)
    al, be = eq.resolve_targets(eq.EquilibrationParams(), A.m, A.n)
    w = eq.objective_weighted(M, u, v, np.full(A.m, al * al), np.full(A.n, be * be), 0.1)
    assert w == pytest.approx(obj, rel=1e-14)
    gw = eq.gradient_weighted(M, u, v, np.full(A.m, al * al), np.full(A.n, be * be), 0.1)
    assert np.array_equal(gw[0], gu) and np.array_equal(gw[1], gv)
    assert np.array_equal(eq.project_box(np.array([-3.0, 0.5, 2.0]), 1.0), [-1.0, 0.5, 1.0])
    with pytest.raises(eq.InvalidArgument, match="bound must be nonnegative"):
        eq.project_box(np.zeros(2), -1.0)
    with pytest.raises(eq.InvalidArgument, match="targets must be positive"):
        eq.rms_error(M, u, v, 0.0, 1.0)


# ---------------------------------------------------------------- degenerate inputs
@pytest.mark.parametrize("m,n,entries", [(4, 3, []), (1, 1, [(0, 0, 2.0)]),
                                         (5, 7, [(4, 6, -1.5)]), (1, 9, [(0, 2, 1.0), (0, 8, 3.0)])])
def test_degenerate_sparse_inputs_vs_oracle(C, m, n, entries):
    """No entries at all, a single entry, one row: SGD and LSQR through the
    CSR and COO constructors agree with the oracle (breakdown included)."""
    rows = np.array([e[0] for e in entries], np.int64)
    cols = np.array([e[1] for e in entries], np.int64)
    vals = np.array([e[2] for e in entries], np.float64)
    rp = np.zeros(m + 1, np.int64)
    np.add.at(rp, rows + 1, 1)
    rp = np.cumsum(rp)
    A = oracle.CsrArrays(m, n, rp, cols.astype(np.int32), vals)
    want = C.sgd_equilibrate(A, iterations=25, seed=3)
    for M in (eq.ExplicitMatrix.from_csr(m, n, rp, cols, vals),
              eq.ExplicitMatrix.sparse(m, n, (rows, cols, vals))):
        got = eq.sgd_equilibrate(M, eq.EquilibrationParams(iterations=25, seed=3))
        for k in "uvde":
            assert np.array_equal(getattr(got, k), getattr(want, k)), k
        b = np.arange(1, m + 1, dtype=np.float64)
        lw = C.lsqr(A, b, 5, 0.0)
        lg = eq.lsqr(M, b, 5, 0.0)
        assert np.array_equal(lg.residual_history, lw.residual_history)
        assert (lg.iterations, lg.breakdown) == (lw.iterations, lw.breakdown)


@pytest.mark.parametrize("case", ["sp", "lr", "c3"])
def test_column_block_rounds_bit_exact(C, golden, monkeypatch, case):
    """Gathered vectors larger than EQUIL_BLOCK_MB are visited in column blocks
    with the row sums carried between launches (engine.cu build_block_layout).
    Forcing tiny blocks here: the trajectory must not change by a bit."""
    monkeypatch.setenv("EQUIL_BLOCK_MB", "0.004")  # 500-coordinate blocks
    if case == "c3":
        from paper_1602_06621_b200 import configs
        inst = configs.config(3, scale=0.02)
        A = oracle.CsrArrays(inst.m, inst.n, inst.row_ptr, inst.col, inst.val)
        want = C.sgd_equilibrate(A, iterations=15, seed=7)
        got = eq.sgd_equilibrate(device_matrix(A), eq.EquilibrationParams(iterations=15, seed=7))
        want = {k: getattr(want, k) for k in "uvde"}
    else:
        A = csr_from_golden(golden, case)
        got = eq.sgd_equilibrate(device_matrix(A), eq.EquilibrationParams(iterations=40, seed=5),
                                 eq.DiagnosticsConfig(stride=10))
        want = {k: golden[f"{case}_sgd_{k}"] for k in "uvde"}
        np.testing.assert_allclose([h.rms for h in got.history], golden[f"{case}_sgd_hist_rms"],
                                   rtol=1e-12, atol=0)
    for k in "uvde":
        assert np.array_equal(getattr(got, k), want[k]), k


# ---------------------------------------------------------------- sharded engine
@pytest.mark.parametrize("p2p", ["1", "0"])
@pytest.mark.parametrize("case,world", [("lr", 2), ("sp", 3), ("c3", 4)])
def test_sharded_engine_bit_identical_via_host_exchange(C, golden, monkeypatch, case, world, p2p):
    """The multi-GPU engine (row shards of A and A^T, padded gathered vectors,
    slot maps, history and LSQR reductions) run as `world` rank handles in one
    process on one GPU, exchanging through the host (EQUIL_HOST_EXCHANGE=1, a
    barrier per exchange; no kernel waits on another rank).  Every rank must
    return the single-GPU result bit for bit, both with the fused all-gather
    (EQUIL_P2P=1: the SGD epilogue stores into every rank's gathered vector)
    and with the padded all-gathers."""
    import os
    import threading
    if case == "c3":
        from paper_1602_06621_b200 import configs
        inst = configs.config(3, scale=0.02)
        A = oracle.CsrArrays(inst.m, inst.n, inst.row_ptr, inst.col, inst.val)
    else:
        A = csr_from_golden(golden, case)
    b = np.random.default_rng(4).standard_normal(A.m)
    p = eq.EquilibrationParams(iterations=20, seed=5)
    d = eq.DiagnosticsConfig(stride=5)
    M1 = device_matrix(A)
    ref_s = eq.sgd_equilibrate(M1, p, d)
    ref_l = eq.lsqr(M1, b, 12, 0.0)
    ref_p = eq.lsqr_preconditioned(M1, b, eq.EquilibrationParams(iterations=8, seed=2), 12, 0.0)
    monkeypatch.setenv("EQUIL_HOST_EXCHANGE", "1")
    monkeypatch.setenv("EQUIL_P2P", p2p)
    nid = os.urandom(128)
    # creation is collective (sharded setup: all-reduce and all-to-all between
    # the ranks), so every rank creates its handle on its own thread
    Ms = [None] * world
    out = [None] * world
    errs = []

    def run(r):
        try:
            Ms[r] = eq.ExplicitMatrix.from_csr(A.m, A.n, A.row_ptr, A.col, A.val, rank=r,
                                               world_size=world, nccl_id=nid)
            s = eq.sgd_equilibrate(Ms[r], p, d)
            lp = eq.lsqr(Ms[r], b, 12, 0.0)
            pp = eq.lsqr_preconditioned(Ms[r], b, eq.EquilibrationParams(iterations=8, seed=2),
                                        12, 0.0)
            out[r] = (s, lp, pp)
        except Exception as ex:  # surfaced below
            errs.append(ex)

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    assert {eq.exchange_mode(M) for M in Ms} == {"p2p" if p2p == "1" else "allgather"}
    for s, lp, pp in out:
        for k in "uvde":
            assert np.array_equal(getattr(s, k), getattr(ref_s, k)), k
        assert (s.box_feasible, s.iterate_bound_ok) == (ref_s.box_feasible, ref_s.iterate_bound_ok)
        assert [h.objective for h in s.history] == [h.objective for h in ref_s.history]
        assert [h.rms for h in s.history] == [h.rms for h in ref_s.history]
        assert np.array_equal(lp.residual_history, ref_l.residual_history)
        assert np.array_equal(lp.x, ref_l.x)
        assert np.array_equal(pp.residual_history, ref_p.residual_history)
        assert np.array_equal(pp.x, ref_p.x)


TRAVERSALS = [
    {},                                                    # interleaved slices (default)
    {"EQUIL_SELL_LONG": "1"},                              # long rows as lane chains
    {"EQUIL_SELL_LONG": "0"},                              # long rows on the staged CTAs
    {"EQUIL_SELL": "0"},                                   # staged traversal throughout
    {"EQUIL_SELL_PASSES": "0"},                            # generic passes staged
    {"EQUIL_SWEEP": "0"},                                  # long rows on the long-slice kernel
    {"EQUIL_SWEEP": "0", "EQUIL_SELL_VARIANT": "1", "EQUIL_SELL_LVARIANT": "3"},
    {"EQUIL_SWEEP": "0", "EQUIL_SELL_VARIANT": "2", "EQUIL_SELL_LVARIANT": "2"},
    {"EQUIL_SWEEP_WIDTH": "300", "EQUIL_SWEEP_STAGES": "3"},  # narrow sweep panels
    {"EQUIL_SELL_ORDER": "1"},                             # warp slices in window order
    {"EQUIL_SELL_QUAD": "0"},                              # every slice 1-wide (no 128/256-bit loads)
    {"EQUIL_SELL_QUAD": "0", "EQUIL_SWEEP": "0"},
    {"EQUIL_SELL_VARIANT": "3"},                           # warp slices at 6 CTAs/SM (80 registers)
    {"EQUIL_SPLIT_EPI": "0"},                              # SGD update fused into the traversals
    {"EQUIL_BLOCK_MB": "0.004"},                           # 500-coordinate column blocks
    {"EQUIL_BLOCK_MB": "0.004", "EQUIL_SELL_BLOCKED": "1"},  # same on interleaved slices
    {"EQUIL_BLOCK_MB": "0.004", "EQUIL_SELL_BLOCKED": "1", "EQUIL_SELL_ORDER": "1"},
]


@pytest.mark.parametrize("env", TRAVERSALS, ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items())
                         or "default")
def test_traversals_bit_exact_on_boundary_row_lengths(C, monkeypatch, env):
    """Every SGD traversal and pass (sell.cu warp slices / warp-specialised
    long slices, their variants, the staged kernels) against the oracle on
    rows whose lengths sit on the boundaries of batches, rounds, the 512-entry
    long-row threshold and partial slices, plus empty rows inside long slices."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    rng = np.random.default_rng(5)
    n = 6000
    lens = [0, 1, 2, 3, 4, 5, 7, 8, 9, 15, 16, 17, 31, 32, 33, 63, 64, 65, 511, 512, 513, 514,
            515, 1000, 1023, 4099, 5999, 6000]
    lens = lens * 3 + list(rng.integers(0, 40, 250)) + [0] * 20
    rng.shuffle(lens)
    m = len(lens)
    cols = [np.sort(rng.choice(n, size=int(L), replace=False)) for L in lens]
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    col = np.concatenate(cols).astype(np.int32)
    val = rng.standard_normal(int(rp[-1])) * np.exp(rng.standard_normal(int(rp[-1])))
    A = oracle.CsrArrays(m, n, rp, col, val)
    M = device_matrix(A)
    w = C.sgd_equilibrate(A, iterations=12, seed=3)
    r = eq.sgd_equilibrate(M, eq.EquilibrationParams(iterations=12, seed=3))
    for k in "uvde":
        assert np.array_equal(getattr(r, k), getattr(w, k)), k
    b = rng.standard_normal(m)
    run = eq.lsqr(M, b, 8, 0.0)
    ref = C.lsqr(A, b, 8, 0.0)
    assert np.array_equal(np.array(run.residual_history), ref.residual_history)
    assert np.array_equal(run.x, ref.x)
    pre = eq.lsqr_preconditioned(M, b, eq.EquilibrationParams(iterations=6, seed=4), 8, 0.0)
    pref = C.lsqr_preconditioned(A, b, 8, 0.0, iterations=6, seed=4)
    assert np.array_equal(np.array(pre.residual_history), pref.residual_history)
    assert np.array_equal(pre.x, pref.x)


def test_one_shot_entry_bit_exact_vs_oracle(C):
    """equil_sgd_equilibrate_csr generates the sign stream while the matrix is
    built (seed and T are known up front): same trajectory as the oracle, and
    invalid parameters still fail with the reference's message."""
    from paper_1602_06621_b200 import configs
    inst = configs.config(1)
    A = oracle.CsrArrays(inst.m, inst.n, inst.row_ptr, inst.col, inst.val)
    for seed, T in [(0, 50), (9, 7), (3, 0)]:
        p = eq.EquilibrationParams(alpha=inst.alpha, beta=inst.beta, iterations=T, seed=seed)
        got = eq.sgd_equilibrate_csr(inst.m, inst.n, inst.row_ptr, inst.col, inst.val, p)
        want = C.sgd_equilibrate(A, alpha=inst.alpha, beta=inst.beta, iterations=T, seed=seed)
        for k in "uvde":
            assert np.array_equal(getattr(got, k), getattr(want, k)), (seed, T, k)
    with pytest.raises(ValueError, match="gamma must be positive"):
        eq.sgd_equilibrate_csr(inst.m, inst.n, inst.row_ptr, inst.col, inst.val,
                               eq.EquilibrationParams(gamma=0.0))


def test_dense_multi_chunk_bit_exact_vs_oracle(C):
    """Dense SGD with several 2048-row and 2048-column chunks (both partial):
    the row and column kernels follow the oracle's canonical order, including
    both level-2 folds."""
    rng = np.random.default_rng(17)
    m, n = 4500, 2600
    a = rng.standard_normal((m, n)) * np.exp(rng.standard_normal((m, 1))) \
        * np.exp(rng.standard_normal((1, n)))
    a[rng.random((m, n)) < 0.01] = 0.0
    A = oracle.CsrArrays(m, n, dense=a)
    p = dict(iterations=4, seed=11)
    w = C.sgd_equilibrate(A, **p)
    r = eq.sgd_equilibrate(device_matrix(A), eq.EquilibrationParams(**p))
    for k in "uvde":
        assert np.array_equal(getattr(r, k), getattr(w, k)), k
