"""Small driver for ncu captures: python tools/ncu_target.py CONFIG T [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1602_06621_b200 as eq  # noqa: E402
from paper_1602_06621_b200 import configs  # noqa: E402


def main():
    k = int(sys.argv[1])
    T = int(sys.argv[2])
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    inst = configs.config(k)
    if inst.dense is not None:
        M = eq.ExplicitMatrix.dense(inst.dense)
    else:
        M = eq.ExplicitMatrix.from_csr(inst.m, inst.n, inst.row_ptr, inst.col, inst.val)
    p = eq.EquilibrationParams(alpha=inst.alpha, beta=inst.beta, iterations=T, seed=inst.seed)
    for _ in range(reps):
        r = eq.sgd_equilibrate(M, p)
    print("ok", float(r.u.sum()), float(r.v.sum()))


if __name__ == "__main__":
    main()
