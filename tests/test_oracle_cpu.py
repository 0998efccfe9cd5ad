"""CPU tests: the oracle (C restatement) pinned against the reference.

Pins, in order of strength:
  * the reference's own KATs (tests/test_sampling.cpp:20-34), the C++
    standard's mt19937_64 KAT, and the survey's probe-stream KATs;
  * golden vectors produced by the reference's own sources
    (tests/golden/ref_golden.npz, see make_golden.py);
  * live comparison with oracle/_ref when the reference tree is present.
"""
import math
import os

import numpy as np
import pytest

import oracle
from conftest import csr_from_golden

CASES = ["sp", "lr", "dn"]


def test_rng_kats_from_reference_tests(C):
    # tests/test_sampling.cpp:20-25
    assert list(C.raw_outputs(42, 0, 0, 3)) == [15474610311340789812, 7401741880442573951,
                                                13284216013538723942]
    assert int(C.raw_outputs(42, 7, 0, 1)[0]) == 16977106985146821793
    # tests/test_sampling.cpp:27-33
    u = C.draws(42, 0, "uniform", 2)
    assert u[0] == pytest.approx(0.83888030589611362, rel=1e-16)
    assert u[1] == pytest.approx(0.40124923134763907, rel=1e-16)
    z = C.draws(42, 0, "normal", 2)
    assert z[0] == pytest.approx(-0.48227979325560744, rel=1e-15)
    assert z[1] == pytest.approx(0.34464574861270958, rel=1e-15)


def test_mt19937_64_standard_kat(C):
    # [rand.predef]: default-seeded mt19937_64's 10000th output
    assert int(C.mt64_std(5489, 10000)[-1]) == 9981545732273789042


def test_probe_stream_kats(C):
    # seeding and probe-stream (stream 17) known answers
    assert C.mixed_seed(0, 17) == 0x97A173C500D33F8D
    assert C.mixed_seed(1, 17) == 0xCC86D3A596A9D8AD
    o = C.raw_outputs(0, 17, 0, 16)
    assert "".join("+" if int(x) >> 63 else "-" for x in o) == "+-----+-+++---+-"
    kat = {0: 0xBD5B2912AF5B876E, 312: 0x5931A92658C55D6A, 5000: 0x2D00AE53818761A1,
           15000: 0x7762068C458255FB}
    for k, v in kat.items():
        assert int(C.raw_outputs(0, 17, k, 1)[0]) == v
    assert int(C.raw_outputs(1, 17, 0, 1)[0]) == 0xEA50F0E7F520213A
    assert int(C.raw_outputs(1, 17, 5000, 1)[0]) == 0xDFD19FC352AD0B83


def test_sign_bits_match_raw_msb(C, golden):
    raw = golden["raw_0_17"]
    bits = C.sign_bits(0, 17, 100, 3000)
    for k in range(3000):
        assert ((bits[k >> 5] >> (k & 31)) & 1) == (int(raw[100 + k]) >> 63)


def test_oracle_rng_matches_golden(C, golden):
    assert np.array_equal(C.raw_outputs(0, 17, 0, 20000), golden["raw_0_17"])
    assert np.array_equal(C.raw_outputs(1, 17, 0, 20000), golden["raw_1_17"])


def test_det_exp_properties(C):
    assert C.L.eo_det_exp(0.0) == 1.0
    x = np.linspace(-20, 20, 4001)
    y = C.det_exp(x)
    rel = np.abs(y - np.exp(x)) / np.exp(x)
    assert rel.max() < 4e-16  # ~1-2 ulp of glibc exp
    assert np.all(np.diff(y) > 0)


def test_canonical_sum_structure(C):
    rng = np.random.default_rng(0)
    for n in [0, 1, 7, 256, 2047, 2048, 2049, 10000, 3 * 2048 * 1024 + 5]:
        x = rng.standard_normal(n)
        s = C.canon_sumsq(x)
        if n:
            assert s == pytest.approx(float(np.sum(x * x)), rel=1e-12)
        else:
            assert s == 0.0
    # explicit restatement of the tree for a small ragged case
    x = rng.standard_normal(2048 + 300)
    def tree(p, lanes):
        s = [0.0] * lanes
        for k, t in enumerate(p):
            s[k % lanes] = s[k % lanes] + t
        h = lanes // 2
        while h >= 1:
            for l in range(h):
                s[l] = s[l] + s[l + h]
            h //= 2
        return s[0]
    parts = [tree(list(x[c:c + 2048] * x[c:c + 2048]), 256) for c in range(0, x.size, 2048)]
    assert C.canon_sumsq(x) == tree(parts, 1024)


@pytest.mark.parametrize("key", CASES)
def test_oracle_matches_reference_golden(C, golden, key):
    A = csr_from_golden(golden, key)
    if A.dense is None:
        T = C.transpose(A)
        assert np.array_equal(T.row_ptr, golden[f"{key}_t_rp"])
        assert np.array_equal(T.col, golden[f"{key}_t_col"])
        assert np.array_equal(T.val, golden[f"{key}_t_val"])
    s = C.sgd_equilibrate(A, iterations=40, seed=5, diag_stride=10)
    for k in "uvde":
        assert np.array_equal(getattr(s, k), golden[f"{key}_sgd_{k}"]), k
    assert np.array_equal(s.hist_rms, golden[f"{key}_sgd_hist_rms"])
    assert np.array_equal(s.hist_objective, golden[f"{key}_sgd_hist_obj"])
    b = golden[f"{key}_b"]
    lp = C.lsqr(A, b, 30, 0.0)
    assert np.array_equal(lp.residual_history, golden[f"{key}_lsqr_res"])
    assert np.array_equal(lp.x, golden[f"{key}_lsqr_x"])
    assert [lp.iterations, lp.reached_tol, lp.breakdown, lp.apply_count,
            lp.adjoint_count] == list(golden[f"{key}_lsqr_meta"])
    pp = C.lsqr_preconditioned(A, b, 30, 0.0, iterations=15, seed=3)
    assert np.array_equal(pp.residual_history, golden[f"{key}_plsqr_res"])
    assert np.array_equal(pp.x, golden[f"{key}_plsqr_x"])
    assert [pp.iterations, pp.reached_tol, pp.breakdown, pp.apply_count,
            pp.adjoint_count] == list(golden[f"{key}_plsqr_meta"])


def test_oracle_targets_variant_matches_reference_golden(C, golden):
    """sgd_equilibrate_targets (src/variants.cpp:105-118) on the oracle vs the
    reference's own sources (golden)."""
    A = csr_from_golden(golden, "sp")
    s = C.sgd_equilibrate_targets(A, golden["tg_r"], golden["tg_c"], iterations=30, seed=4,
                                  diag_stride=10)
    for k in "uvde":
        assert np.array_equal(getattr(s, k), golden[f"tg_sgd_{k}"])
    assert np.array_equal(s.hist_objective, golden["tg_sgd_hist_obj"])
    # uniform targets reproduce sgd_equilibrate bit for bit (test_variants.cpp:97-110)
    al = (A.n / A.m) ** 0.25
    be = (A.m / A.n) ** 0.25
    a, b = C.sgd_equilibrate(A, iterations=40, seed=5), C.sgd_equilibrate_targets(
        A, np.full(A.m, al * al), np.full(A.n, be * be), iterations=40, seed=5)
    import math
    if (al, be) == (math.pow(A.n / A.m, 0.25), math.pow(A.m / A.n, 0.25)):
        for k in "uvde":
            assert np.array_equal(getattr(a, k), getattr(b, k))


@pytest.mark.skipif(not oracle.ref_available(), reason="reference sources absent")
def test_oracle_matches_live_reference_random():
    """Live: C restatement vs the reference's own sources on fresh inputs."""
    C, R = oracle.c_oracle(), oracle.ref_oracle()
    rng = np.random.default_rng(7)
    for m, n, dens, T, seed in [(60, 90, 0.1, 30, 0), (120, 40, 0.2, 25, 9), (1, 1, 1.0, 10, 2)]:
        mask = rng.random((m, n)) < dens
        mask[0, 0] = True
        a = rng.standard_normal((m, n)) * np.exp(rng.standard_normal((m, 1)))
        rp = np.concatenate([[0], np.cumsum(mask.sum(1))])
        A = oracle.CsrArrays(m, n, rp, np.nonzero(mask)[1], a[mask])
        RM = R.matrix(A)
        s1 = C.sgd_equilibrate(A, iterations=T, seed=seed, diag_stride=3)
        s2 = RM.sgd_equilibrate(iterations=T, seed=seed, diag_stride=3)
        for k in "uvde":
            assert np.array_equal(getattr(s1, k), getattr(s2, k))
        assert (s1.box_feasible, s1.iterate_bound_ok) == (s2.box_feasible, s2.iterate_bound_ok)
        b = rng.standard_normal(m)
        assert np.array_equal(C.lsqr(A, b, 20, 0.0).residual_history,
                              RM.lsqr(b, 20, 0.0).residual_history)


def test_reference_known_answers_on_oracle(C):
    """test_equilibrate.cpp:183-227 and :302-331 restated on the oracle."""
    eye = oracle.CsrArrays(5, 5, np.arange(6), np.arange(5), np.ones(5))
    s = C.sgd_equilibrate(eye, alpha=1.0, beta=1.0, iterations=50, diag_stride=1)
    assert np.all(s.u == 0) and np.all(s.v == 0) and np.all(s.d == 1) and np.all(s.e == 1)
    assert np.allclose(s.hist_objective, 2.5, rtol=1e-15)
    assert np.allclose(s.hist_rms, 0.0, atol=1e-15)
    # 1x1 [2]: projected GD to the scalar stationarity root (-0.338)
    one = oracle.CsrArrays(1, 1, dense=np.array([[2.0]]))
    s = C.sgd_equilibrate(one, alpha=1.0, beta=1.0, gamma=0.1, max_log_scale=10.0,
                          iterations=10000)
    assert abs(s.u[0] + 0.338) < 2e-3 + 1e-3 and abs(s.v[0] + 0.338) < 3e-3
    # zero matrix: the average carries weights 2(t+1)/((T+1)(T+2))
    z = oracle.CsrArrays(1, 1, dense=np.zeros((1, 1)))
    T, M = 57, 9.210340371976184
    s = C.sgd_equilibrate(z, alpha=1.0, beta=1.0, iterations=T)
    x, it = 0.0, [0.0]
    for t in range(1, T + 1):
        x = min(max(x - 2.0 / (0.1 * (t + 1)) * (0.0 - 1.0 + 0.1 * x), -M), M)
        it.append(x)
    w = [2.0 * (t + 1) / ((T + 1) * (T + 2)) for t in range(T + 1)]
    assert s.u[0] == pytest.approx(sum(a * b for a, b in zip(w, it)), rel=1e-13)


def test_oracle_errors(C):
    A = oracle.CsrArrays(2, 2, np.array([0, 1, 2]), np.array([0, 1]), np.array([1.0, 1.0]))
    with pytest.raises(oracle.OracleError, match="gamma"):
        C.sgd_equilibrate(A, gamma=0.0, iterations=1)
    with pytest.raises(oracle.OracleError, match="alpha"):
        C.sgd_equilibrate(A, alpha=1.0, beta=2.0, iterations=1)
    with pytest.raises(oracle.OracleError, match="nonzero"):
        C.lsqr(A, np.zeros(2), 5, 0.0)


def test_oracle_symmetric_and_block_variants_match_reference_golden(C, golden):
    """sgd_equilibrate_symmetric (src/variants.cpp:35-103) and
    sgd_equilibrate_block (:156-240) on the oracle vs the reference's own
    sources (golden), history included."""
    S = csr_from_golden(golden, "sy")
    s = C.sgd_equilibrate_symmetric(S, iterations=40, seed=6, diag_stride=10)
    for k in "uvde":
        assert np.array_equal(getattr(s, k), golden[f"sy_sgd_{k}"]), k
    assert np.array_equal(s.hist_objective, golden["sy_sgd_hist_obj"])
    assert np.array_equal(s.hist_rms, golden["sy_sgd_hist_rms"])
    assert [s.box_feasible, s.iterate_bound_ok, s.apply_count, s.adjoint_count] == \
        list(golden["sy_sgd_flags"])
    A = csr_from_golden(golden, "sp")
    rb, cb = golden["bl_rb"], golden["bl_cb"]
    b = C.sgd_equilibrate_block(A, rb, cb, 17, int(cb.max()) + 1, iterations=30, seed=8,
                                diag_stride=10)
    for k in "uvde":
        assert np.array_equal(getattr(b, k), golden[f"bl_sgd_{k}"]), k
    assert np.array_equal(b.hist_objective, golden["bl_sgd_hist_obj"])
    assert np.array_equal(b.hist_rms, golden["bl_sgd_hist_rms"])


def test_oracle_variant_known_answers(C):
    """test_variants.cpp:36-61, :165-176, :234-249 restated on the oracle."""
    eye = oracle.CsrArrays(4, 4, np.arange(5), np.arange(4), np.ones(4))
    s = C.sgd_equilibrate_symmetric(eye, alpha=1.0, beta=1.0, iterations=100)
    assert np.all(s.u == 0) and np.array_equal(s.u, s.v) and np.array_equal(s.d, s.e)
    assert (s.apply_count, s.adjoint_count) == (100, 0)
    rng = np.random.default_rng(61)
    ns = oracle.CsrArrays(5, 5, dense=rng.standard_normal((5, 5)))
    with pytest.raises(oracle.OracleError, match="symmetry check"):
        C.sgd_equilibrate_symmetric(ns, alpha=1.0, beta=1.0, iterations=5)
    with pytest.raises(oracle.OracleError, match="must be square"):
        C.sgd_equilibrate_symmetric(oracle.CsrArrays(3, 4, dense=np.ones((3, 4))), alpha=1.0,
                                    beta=1.0, iterations=5)
    A = oracle.CsrArrays(5, 7, dense=rng.standard_normal((5, 7)))
    plain = C.sgd_equilibrate(A, iterations=300, seed=11)
    blk = C.sgd_equilibrate_block(A, np.arange(5), np.arange(7), 5, 7, iterations=300, seed=11)
    for k in "uvde":
        assert np.array_equal(getattr(plain, k), getattr(blk, k))
    B = oracle.CsrArrays(3, 2, dense=rng.standard_normal((3, 2)) + 1.5)
    for rb, cb, R, Cb, msg in [([0, 0, 1], [0, 1], 3, 2, "empty row block"),
                               ([0, 0, 1], [0, 1], 1, 2, "row block index out of range"),
                               ([0, 0, 1], [0, -1], 2, 2, "col block index out of range"),
                               ([0, 0, 1], [0, 1], 0, 2, "block counts must be positive")]:
        with pytest.raises(oracle.OracleError, match=msg):
            C.sgd_equilibrate_block(B, rb, cb, R, Cb, iterations=3)
    one = C.sgd_equilibrate_block(B, [0, 0, 0], [0, 0], 1, 1, iterations=50)
    assert one.u[0] == one.u[1] == one.u[2] and one.v[0] == one.v[1]


@pytest.mark.parametrize("key", ["sp", "dn"])
def test_oracle_ccp_and_spectral_norm_match_reference_golden(C, golden, key):
    """spectral_norm (src/lsqr.cpp:140-163) and ccp_lasso(_preconditioned)
    (src/ccp.cpp:27-141) on the oracle vs the reference's own sources."""
    A = csr_from_golden(golden, key)
    b = golden[f"{key}_b"]
    sn = golden[f"{key}_snorm"]
    assert C.spectral_norm(A, 100, 1e-9, 0) == sn[0]
    assert C.spectral_norm(A, 300, 1e-12, 1) == sn[1]
    ps = float(golden[f"{key}_pstar"][0])
    for tag, kw in [("ccp", dict(max_iters=150)),
                    ("pccp", dict(max_iters=150, params=dict(iterations=30, seed=3))),
                    ("eccp", dict(max_iters=20000, gap_tol=1e-4))]:
        r = C.ccp_lasso(A, b, 0.3, p_star=ps, **kw)
        assert np.array_equal(r.x, golden[f"{key}_{tag}_x"]), tag
        assert np.array_equal(r.objective_history, golden[f"{key}_{tag}_obj"]), tag
        assert np.array_equal(r.gap_history, golden[f"{key}_{tag}_gap"]), tag
        assert [r.iterations, r.equil_iterations, r.reached_tol, r.apply_count,
                r.adjoint_count] == list(golden[f"{key}_{tag}_meta"]), tag
        assert [r.tau, r.sigma, r.theta] == list(golden[f"{key}_{tag}_steps"]), tag


def test_oracle_ccp_known_answers(C):
    """test_itersolvers.cpp:173-227, :273-292 restated on the oracle."""
    D = oracle.CsrArrays(2, 2, dense=np.diag([3.0, 1.0]))
    assert C.spectral_norm(D, 500, 1e-12) == pytest.approx(3.0, rel=1e-8)
    eye = oracle.CsrArrays(2, 2, np.arange(3), np.arange(2), np.ones(2))
    b = np.array([3.0, 0.0])
    assert C.lasso_objective(eye, b, 4.0, np.zeros(2)) == pytest.approx(4.5, rel=1e-14)
    assert C.lasso_objective(eye, b, 4.0, np.array([1.0, 0.0])) == pytest.approx(4.0, rel=1e-14)
    r = C.ccp_lasso(eye, b, 4.0, max_iters=5000)
    assert r.x[0] == pytest.approx(1.0, rel=1e-6) and abs(r.x[1]) <= 1e-8
    assert len(r.objective_history) == r.iterations + 1
    assert r.apply_count == r.adjoint_count == r.iterations
    assert r.tau * r.sigma <= 0.81 + 1e-12
    rng = np.random.default_rng(91)
    A = oracle.CsrArrays(10, 14, dense=rng.standard_normal((10, 14)))
    bb = rng.standard_normal(10)
    plain = C.ccp_lasso(A, bb, 0.05, max_iters=500)
    pre = C.ccp_lasso(A, bb, 0.05, max_iters=500, params=dict(iterations=0))
    assert pre.equil_iterations == 0 and np.array_equal(pre.x, plain.x)
    assert np.array_equal(pre.objective_history, plain.objective_history)
    with pytest.raises(oracle.OracleError, match="lambda must be positive"):
        C.ccp_lasso(A, bb, 0.0, max_iters=5)
    with pytest.raises(oracle.OracleError, match="rhs must be nonzero"):
        C.ccp_lasso(A, np.zeros(10), 0.1, max_iters=5)
    with pytest.raises(oracle.OracleError, match="max_iters must be nonnegative"):
        C.ccp_lasso(A, bb, 0.1, max_iters=-1)


@pytest.mark.parametrize("key", ["sp", "dn"])
def test_oracle_helpers_match_reference_golden(C, golden, key):
    """stochastic_gradient_estimate (src/equilibrate.cpp:60-71) bit-exact; the
    objective and rms_error restatements to 1e-12 (the reference uses std::exp
    and plain sequential sums, src/equilibrate.cpp:10-22, metrics.cpp:24-56)."""
    A = csr_from_golden(golden, key)
    u, v = golden[f"{key}_hu"], golden[f"{key}_hv"]
    su, sv = C.stochastic_gradient_estimate(A, u, v, 7, 17, 123)
    assert np.array_equal(su, golden[f"{key}_hsu"]) and np.array_equal(sv, golden[f"{key}_hsv"])
    a2 = (A.n / A.m) ** 0.5  # alpha^2 for auto targets
    obj = C.objective(A, u, v, a2, (A.m / A.n) ** 0.5, 0.1)
    assert obj == pytest.approx(golden[f"{key}_hobj"][0], rel=1e-12)
    assert C.rms_error(A, u, v, 0.7, 1.1) == pytest.approx(golden[f"{key}_hrms"][0], rel=1e-12)
