"""Quick GPU timing probe (development aid, not the bench contract)."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(
    __import__("os").path.abspath(__file__))))
import paper_1602_06621_b200 as eq  # noqa: E402
from paper_1602_06621_b200 import _lib, configs  # noqa: E402


def time_sgd(M, p, reps=5):
    L = _lib.load()
    s = torch.cuda.ExternalStream(L.equil_matrix_stream(M._h))
    eq.sgd_equilibrate(M, p)  # warm (graph capture)
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        eq.sgd_equilibrate(M, p)
        e1.record(s)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    return min(ts), ts


def main():
    which = sys.argv[1:] or ["1", "2", "3"]
    res = {}
    for k in which:
        k = int(k)
        if k == 4:  # LSQR on c3 (config 4): per-iteration time, plain and preconditioned
            inst = configs.config(4)
            b = configs.rhs(inst)
            M = eq.ExplicitMatrix.from_csr(inst.m, inst.n, inst.row_ptr, inst.col, inst.val)
            out = {}
            for name, fn in [("lsqr", lambda it: eq.lsqr(M, b, it, 0.0)),
                             ("lsqr_pre", lambda it: eq.lsqr_preconditioned(
                                 M, b, eq.EquilibrationParams(iterations=50), it, 0.0))]:
                fn(5)
                t0 = time.perf_counter()
                r10 = fn(10)
                t1 = time.perf_counter()
                r110 = fn(110)
                t2 = time.perf_counter()
                out[name] = {"ms_per_lsqr_iter": ((t2 - t1) - (t1 - t0)) / 100 * 1e3,
                             "final_residual_110": r110.residual_history[-1]}
            print(json.dumps({4: out}), flush=True)
            del M
            continue
        t0 = time.time()
        inst = configs.config(k)
        tg = time.time() - t0
        t0 = time.time()
        if inst.dense is not None:
            M = eq.ExplicitMatrix.dense(inst.dense)
        else:
            M = eq.ExplicitMatrix.from_csr(inst.m, inst.n, inst.row_ptr, inst.col, inst.val)
        torch.cuda.synchronize()
        tc = time.time() - t0
        p = eq.EquilibrationParams(alpha=inst.alpha, beta=inst.beta, iterations=inst.iterations,
                                   seed=inst.seed)
        best, ts = time_sgd(M, p)
        T = inst.iterations
        nnz, m, n = inst.nnz, inst.m, inst.n
        if inst.dense is not None:
            B = 8 * m * n + 48.125 * (m + n)
        else:
            B = 24 * nnz + 52.125 * (m + n)
        res[k] = dict(m=m, n=n, nnz=nnz, gen_s=tg, create_s=tc, call_s=best,
                      ms_per_iter=best / T * 1e3, iters_per_s=T / best,
                      alg_GBps=B * T / best / 1e9, all=ts)
        print(json.dumps({k: res[k]}), flush=True)
        del M


if __name__ == "__main__":
    main()
