"""Full-size parity fixtures (BASELINE configs 3 and 4) from the oracle AND the
reference's own sources.

The GPU box has no /root/reference and the oracle needs minutes per run at
these sizes, so the results are committed as small JSON files here and the
GPU tests / bench.py compare against them:

  fullsize_c3.json     config 3 (2e6 x 1e6, nnz 1.535e8), sgd_equilibrate T=100
                       seed 0: SHA-256 of u, v, d, e (+ heads), flags, counts
  fullsize_c4p.json    config 4 plain lsqr, 500 iterations, tol 0: the whole
                       residual history (exact, float.hex) and SHA-256 of x
  fullsize_c4q.json    config 4 lsqr_preconditioned, T=50, 500 iterations
  fullsize_c3h.json    config 3, T=20 with diagnostics every 5 iterations: the
                       per-iteration objective and RMS row/column-norm spread
                       (src/equilibrate.cpp:174-195, src/metrics.cpp:24-56)

Each part is computed twice, by the C restatement (oracle/liboracle.so) and by
the reference's own translation units (oracle/_ref/libequil_ref.so, built
unmodified from /root/reference/proj/src; src/equilibrate.cpp:138-221,
src/lsqr.cpp:85-138), and the script refuses to write a fixture unless both
agree bit for bit.  Parts run as separate processes so they can go in
parallel:

    python tests/golden/make_fullsize.py c3 oracle   # -> /tmp/fs_c3_oracle.json
    python tests/golden/make_fullsize.py c3 ref
    python tests/golden/make_fullsize.py c4p oracle  # ... c4p ref, c4q oracle, c4q ref
    python tests/golden/make_fullsize.py merge       # -> tests/golden/fullsize_*.json
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

HERE = os.path.dirname(os.path.abspath(__file__))
T_C3, T_C4, LSQR_ITERS = 100, 50, 500


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def instance_digest(inst) -> dict:
    return {"m": inst.m, "n": inst.n, "nnz": inst.nnz, "row_ptr": sha(inst.row_ptr),
            "col": sha(inst.col), "val": sha(inst.val)}


def scaling_record(r) -> dict:
    out = {k: sha(getattr(r, k)) for k in "uvde"}
    out["head"] = {k: [float(x).hex() for x in getattr(r, k)[:4]] for k in "uvde"}
    out.update(alpha=float(r.alpha).hex(), beta=float(r.beta).hex(),
               box_feasible=bool(r.box_feasible), iterate_bound_ok=bool(r.iterate_bound_ok),
               apply_count=int(r.apply_count), adjoint_count=int(r.adjoint_count))
    return out


def lsqr_record(run) -> dict:
    return {"residual_history": [float(x).hex() for x in run.residual_history],
            "x": sha(run.x), "x_head": [float(x).hex() for x in run.x[:4]],
            "iterations": int(run.iterations), "reached_tol": bool(run.reached_tol),
            "breakdown": bool(run.breakdown), "apply_count": int(run.apply_count),
            "adjoint_count": int(run.adjoint_count)}


def run_part(part: str, who: str) -> dict:
    import oracle
    from paper_1602_06621_b200 import configs
    t0 = time.time()
    inst = configs.config(3 if part in ("c3", "c3h") else 4)
    A = oracle.CsrArrays(inst.m, inst.n, inst.row_ptr, inst.col, inst.val)
    rec = {"instance": instance_digest(inst), "who": who}
    if who == "ref":
        R = oracle.ref_oracle()
        M = R.matrix(A)
    else:
        Co = oracle.c_oracle()
    t1 = time.time()
    if part == "c3":
        rec["config"] = {"iterations": T_C3, "seed": 0, "alpha": "auto", "beta": "auto"}
        r = (M.sgd_equilibrate(iterations=T_C3, seed=0) if who == "ref"
             else Co.sgd_equilibrate(A, iterations=T_C3, seed=0))
        rec["result"] = scaling_record(r)
    elif part == "c3h":
        rec["config"] = {"iterations": 20, "seed": 0, "diag_stride": 5}
        r = (M.sgd_equilibrate(iterations=20, seed=0, diag_stride=5) if who == "ref"
             else Co.sgd_equilibrate(A, iterations=20, seed=0, diag_stride=5))
        rec["result"] = scaling_record(r)
        # diagnostics do not feed back; compared at 1e-12 relative,
        # so the two implementations are recorded separately
        rec["history"] = {"iter": [int(x) for x in r.hist_iter],
                          "objective": [float(x).hex() for x in r.hist_objective],
                          "rms": [float(x).hex() for x in r.hist_rms]}
    else:
        b = configs.rhs(inst)
        rec["b"] = sha(b)
        rec["config"] = {"max_iters": LSQR_ITERS, "tol": 0.0, "seed": 0}
        if part == "c4p":
            run = M.lsqr(b, LSQR_ITERS, 0.0) if who == "ref" else Co.lsqr(A, b, LSQR_ITERS, 0.0)
        else:
            rec["config"]["iterations"] = T_C4
            run = (M.lsqr_preconditioned(b, LSQR_ITERS, 0.0, iterations=T_C4, seed=0)
                   if who == "ref" else
                   Co.lsqr_preconditioned(A, b, LSQR_ITERS, 0.0, iterations=T_C4, seed=0))
        rec["result"] = lsqr_record(run)
    rec["seconds"] = {"setup": round(t1 - t0, 1), "run": round(time.time() - t1, 1)}
    return rec


def merge() -> None:
    names = {"c3": "fullsize_c3.json", "c3h": "fullsize_c3h.json",
             "c4p": "fullsize_c4p.json", "c4q": "fullsize_c4q.json"}
    for part, name in names.items():
        recs = {}
        for who in ("oracle", "ref"):
            p = f"/tmp/fs_{part}_{who}.json"
            if os.path.exists(p):
                with open(p) as f:
                    recs[who] = json.load(f)
        if len(recs) != 2:
            print(f"{part}: missing {set(('oracle', 'ref')) - set(recs)}; skipped")
            continue
        a, b = recs["oracle"], recs["ref"]
        for k in ("instance", "config", "result"):
            if a[k] != b[k]:
                raise SystemExit(f"{part}: oracle and reference differ in {k}")
        if a.get("b") != b.get("b"):
            raise SystemExit(f"{part}: rhs differs")
        out = {k: a[k] for k in ("instance", "config", "result") if k in a}
        if "history" in a:
            ha = [float.fromhex(x) for x in a["history"]["objective"] + a["history"]["rms"]]
            hb = [float.fromhex(x) for x in b["history"]["objective"] + b["history"]["rms"]]
            if a["history"]["iter"] != b["history"]["iter"] or any(
                    abs(x - y) > 1e-12 * max(abs(x), abs(y)) for x, y in zip(ha, hb)):
                raise SystemExit(f"{part}: histories differ beyond 1e-12")
            out["history"] = a["history"]
            out["history_reference"] = b["history"]
        if "b" in a:
            out["b"] = a["b"]
        out["generated_by"] = ("tests/golden/make_fullsize.py: oracle/liboracle.so and "
                               "oracle/_ref/libequil_ref.so agree bit for bit")
        out["cpu_seconds"] = {"oracle": a["seconds"], "reference": b["seconds"]}
        with open(os.path.join(HERE, name), "w") as f:
            json.dump(out, f, indent=1)
        print("wrote", name)


if __name__ == "__main__":
    if sys.argv[1] == "merge":
        merge()
    else:
        part, who = sys.argv[1], sys.argv[2]
        rec = run_part(part, who)
        with open(f"/tmp/fs_{part}_{who}.json", "w") as f:
            json.dump(rec, f)
        print(part, who, rec["seconds"])
