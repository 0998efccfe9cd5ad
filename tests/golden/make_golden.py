"""Generate tests/golden/ref_golden.npz from the REFERENCE's own sources.

Runs oracle/_ref/libequil_ref.so (the reference's hot-path translation units
compiled unmodified against oracle/eigen_lite; see oracle/Makefile) in this
container, where /root/reference exists.  The GPU box has no /root/reference,
so the fixtures are committed and the GPU tests read them.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ref_golden.npz")


def badly_scaled_sparse(m, n, density, seed):
    rng = np.random.default_rng(seed)
    mask = rng.random((m, n)) < density
    a = rng.standard_normal((m, n)) * np.exp(rng.standard_normal((m, 1))) \
        * np.exp(rng.standard_normal((1, n)))
    rows, cols = np.nonzero(mask)
    rp = np.concatenate([[0], np.cumsum(mask.sum(1))]).astype(np.int64)
    return oracle.CsrArrays(m, n, rp, cols.astype(np.int32), a[mask])


def long_row_sparse(seed):
    """rows/columns longer than one 2048-entry tile, empty rows and columns"""
    rng = np.random.default_rng(seed)
    m, n = 700, 5000
    lens = rng.integers(0, 12, m)
    lens[[3, 100, 650]] = [4500, 2049, 2048]
    lens[[5, 6, 7]] = 0
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    cols = []
    for L in lens:
        c = np.sort(rng.choice(n - 10, size=L, replace=False))  # last 10 columns empty
        cols.append(c)
    col = np.concatenate(cols).astype(np.int32)
    # make column 17 long in A^T too
    val = rng.standard_normal(col.size) * np.exp(rng.standard_normal(col.size))
    return oracle.CsrArrays(m, n, rp, col, val)


def main():
    R = oracle.ref_oracle()
    g = {}
    # ---- RNG: test_sampling.cpp:20-25 KATs plus probe-stream sign bits
    g["kat_42_0"] = R.outputs(42, 0, 3)
    g["kat_42_7"] = R.outputs(42, 7, 1)
    g["raw_0_17"] = R.outputs(0, 17, 20000)
    g["raw_1_17"] = R.outputs(1, 17, 20000)

    cases = {
        "sp": badly_scaled_sparse(300, 200, 0.03, 11),
        "lr": long_row_sparse(12),
        "dn": None,
    }
    rng = np.random.default_rng(13)
    dense = rng.standard_normal((40, 25)) * np.exp(2 * rng.standard_normal((40, 1)))
    cases["dn"] = oracle.CsrArrays(40, 25, dense=dense)
    for key, A in cases.items():
        g[f"{key}_shape"] = np.array([A.m, A.n])
        if A.dense is not None:
            g[f"{key}_dense"] = A.dense
        else:
            g[f"{key}_rp"], g[f"{key}_col"], g[f"{key}_val"] = A.row_ptr, A.col, A.val
        RM = R.matrix(A)
        if A.dense is None:
            T = RM.transposed().export()
            g[f"{key}_t_rp"], g[f"{key}_t_col"], g[f"{key}_t_val"] = T.row_ptr, T.col, T.val
        s = RM.sgd_equilibrate(iterations=40, seed=5, diag_stride=10)
        for k in "uvde":
            g[f"{key}_sgd_{k}"] = getattr(s, k)
        g[f"{key}_sgd_hist_rms"] = s.hist_rms
        g[f"{key}_sgd_hist_obj"] = s.hist_objective
        g[f"{key}_sgd_flags"] = np.array([s.box_feasible, s.iterate_bound_ok,
                                          s.apply_count, s.adjoint_count])
        b = np.random.default_rng(14).standard_normal(A.m)
        g[f"{key}_b"] = b
        lp = RM.lsqr(b, 30, 0.0)
        g[f"{key}_lsqr_res"], g[f"{key}_lsqr_x"] = lp.residual_history, lp.x
        g[f"{key}_lsqr_meta"] = np.array([lp.iterations, lp.reached_tol, lp.breakdown,
                                          lp.apply_count, lp.adjoint_count])
        pp = RM.lsqr_preconditioned(b, 30, 0.0, iterations=15, seed=3)
        g[f"{key}_plsqr_res"], g[f"{key}_plsqr_x"] = pp.residual_history, pp.x
        g[f"{key}_plsqr_meta"] = np.array([pp.iterations, pp.reached_tol, pp.breakdown,
                                           pp.apply_count, pp.adjoint_count])
    # nonuniform targets (src/variants.cpp:105-118) on the sparse case
    A = cases["sp"]
    rng = np.random.default_rng(15)
    r = rng.uniform(0.5, 2.0, A.m)
    c = rng.uniform(0.5, 2.0, A.n)
    c = c * (r.sum() / c.sum())
    s = R.matrix(A).sgd_equilibrate_targets(r, c, iterations=30, seed=4, diag_stride=10)
    g["tg_r"], g["tg_c"] = r, c
    for k in "uvde":
        g[f"tg_sgd_{k}"] = getattr(s, k)
    g["tg_sgd_hist_obj"] = s.hist_objective
    g["tg_sgd_flags"] = np.array([s.box_feasible, s.iterate_bound_ok, s.apply_count,
                                  s.adjoint_count])
    # symmetric variant (src/variants.cpp:35-103) on an exactly symmetric matrix
    rng = np.random.default_rng(16)
    ns = 120
    mask = rng.random((ns, ns)) < 0.05
    mask |= mask.T
    np.fill_diagonal(mask, True)
    sc = np.exp(rng.standard_normal(ns))
    a = rng.standard_normal((ns, ns)) * sc[:, None] * sc[None, :]
    a = np.triu(a) + np.triu(a, 1).T
    rows, cols = np.nonzero(mask)
    S = oracle.CsrArrays(ns, ns, np.concatenate([[0], np.cumsum(mask.sum(1))]).astype(np.int64),
                         cols.astype(np.int32), a[mask])
    g["sy_shape"] = np.array([ns, ns])
    g["sy_rp"], g["sy_col"], g["sy_val"] = S.row_ptr, S.col, S.val
    s = R.matrix(S).sgd_equilibrate_symmetric(iterations=40, seed=6, diag_stride=10)
    for k in "uvde":
        g[f"sy_sgd_{k}"] = getattr(s, k)
    g["sy_sgd_hist_obj"], g["sy_sgd_hist_rms"] = s.hist_objective, s.hist_rms
    g["sy_sgd_flags"] = np.array([s.box_feasible, s.iterate_bound_ok, s.apply_count,
                                  s.adjoint_count])
    # block variant (src/variants.cpp:156-240) on the sparse case
    A = cases["sp"]
    rb = rng.integers(0, 17, A.m)
    rb[:17] = np.arange(17)
    cb = np.arange(A.n) // 9
    s = R.matrix(A).sgd_equilibrate_block(rb, cb, 17, int(cb.max()) + 1, iterations=30, seed=8,
                                          diag_stride=10)
    g["bl_rb"], g["bl_cb"] = rb, cb
    for k in "uvde":
        g[f"bl_sgd_{k}"] = getattr(s, k)
    g["bl_sgd_hist_obj"], g["bl_sgd_hist_rms"] = s.hist_objective, s.hist_rms
    g["bl_sgd_flags"] = np.array([s.box_feasible, s.iterate_bound_ok, s.apply_count,
                                  s.adjoint_count])
    # spectral_norm (src/lsqr.cpp:140-163) and the Chambolle-Pock lasso
    # (src/ccp.cpp): plain, preconditioned, early stop on the gap
    for key in ["sp", "dn"]:
        A = cases[key]
        RM = R.matrix(A)
        b = g[f"{key}_b"]
        g[f"{key}_snorm"] = np.array([RM.spectral_norm(100, 1e-9, 0),
                                      RM.spectral_norm(300, 1e-12, 1)])
        lam = 0.3
        xf, ps = RM.lasso_fista(b, lam, 1e-10, 200000)
        g[f"{key}_pstar"] = np.array([ps])
        for tag, kw in [("ccp", dict(max_iters=150)),
                        ("pccp", dict(max_iters=150, params=dict(iterations=30, seed=3))),
                        ("eccp", dict(max_iters=20000, gap_tol=1e-4))]:
            r = RM.ccp_lasso(b, lam, p_star=ps, **kw)
            g[f"{key}_{tag}_x"] = r.x
            g[f"{key}_{tag}_obj"] = r.objective_history
            g[f"{key}_{tag}_gap"] = r.gap_history
            g[f"{key}_{tag}_meta"] = np.array([r.iterations, r.equil_iterations, r.reached_tol,
                                               r.apply_count, r.adjoint_count])
            g[f"{key}_{tag}_steps"] = np.array([r.tau, r.sigma, r.theta])
    # equilibrate.hpp / metrics.hpp helpers at a fixed (u, v): objective, gradient,
    # rms_error (std::exp and sequential sums: tolerance references) and the
    # stochastic gradient estimate (bit-exact reference)
    for key in ["sp", "dn"]:
        A = cases[key]
        RM = R.matrix(A)
        rng = np.random.default_rng(17)
        u, v = 0.3 * rng.standard_normal(A.m), 0.3 * rng.standard_normal(A.n)
        g[f"{key}_hu"], g[f"{key}_hv"] = u, v
        g[f"{key}_hobj"] = np.array([RM.objective(u, v), RM.objective(u, v, 0.9, 0.0, 0.3)])
        gu, gv = RM.gradient(u, v)
        g[f"{key}_hgu"], g[f"{key}_hgv"] = gu, gv
        g[f"{key}_hrms"] = np.array([RM.rms_error(u, v, 0.7, 1.1)])
        su, sv = RM.stochastic_gradient_estimate(u, v, 7, 17, 123)
        g[f"{key}_hsu"], g[f"{key}_hsv"] = su, sv
    np.savez_compressed(OUT, **g)
    print(OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
