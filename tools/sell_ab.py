"""A/B of SGD traversals on one matrix (development aid, not the bench contract).

    python tools/sell_ab.py [config] [spec ...]

Each spec is ENV=VAL[,ENV=VAL...] applied before the matrix is created, e.g.
EQUIL_SELL=0  EQUIL_SELL_VARIANT=2.  Prints ms per iteration (live events
around the graph's T loop, best of 3 calls) and whether u, v, d, e equal the
first spec's bit for bit.
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1602_06621_b200 as eq  # noqa: E402
from paper_1602_06621_b200 import configs  # noqa: E402


def main():
    k = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    specs = sys.argv[2:] or ["EQUIL_SELL=0", "EQUIL_SELL=1"]
    inst = configs.config(k)
    p = eq.EquilibrationParams(alpha=inst.alpha, beta=inst.beta, iterations=inst.iterations,
                               seed=inst.seed)
    ref = None
    for spec in specs:
        saved = {}
        for kv in spec.split(","):
            key, val = kv.split("=", 1)
            saved[key] = os.environ.get(key)
            os.environ[key] = val
        M = eq.ExplicitMatrix.from_csr(inst.m, inst.n, inst.row_ptr, inst.col, inst.val)
        r = eq.sgd_equilibrate(M, p)
        best = 1e30
        for _ in range(3):
            r = eq.sgd_equilibrate(M, p)
            ms, it = eq.last_loop_ms(M)
            best = min(best, ms / max(it, 1))
        same = None
        if ref is None:
            ref = r
        else:
            same = all(np.array_equal(getattr(r, q), getattr(ref, q)) for q in "uvde")
        print(json.dumps({"spec": spec, "ms_per_iter": round(best, 4), "bit_identical": same}),
              flush=True)
        M.close()
        for key, v in saved.items():
            if v is None:
                os.environ.pop(key, None)
            else:
                os.environ[key] = v


if __name__ == "__main__":
    main()
