"""One rank of tests/test_gpu_multiprocess.py: a separate PROCESS that builds
its shard of a sharded matrix (EQUIL_HOST_EXCHANGE=2: POSIX shared-memory host
exchange, peers' gathered-vector buffers mapped with cudaIpcOpenMemHandle),
runs sgd_equilibrate / lsqr / lsqr_preconditioned, and saves what it got.

    python tests/_mp_worker.py RANK WORLD ID_HEX OUT.npz
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1602_06621_b200 as eq  # noqa: E402
from paper_1602_06621_b200 import configs  # noqa: E402


def main():
    rank, world, idhex, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4]
    inst = configs.config(3, scale=0.02)
    b = np.random.default_rng(4).standard_normal(inst.m)
    M = eq.ExplicitMatrix.from_csr(inst.m, inst.n, inst.row_ptr, inst.col, inst.val,
                                   rank=rank, world_size=world, nccl_id=bytes.fromhex(idhex))
    s = eq.sgd_equilibrate(M, eq.EquilibrationParams(iterations=20, seed=5),
                           eq.DiagnosticsConfig(stride=5))
    mode = eq.exchange_mode(M)
    lp = eq.lsqr(M, b, 12, 0.0)
    pp = eq.lsqr_preconditioned(M, b, eq.EquilibrationParams(iterations=8, seed=2), 12, 0.0)
    np.savez(out, u=s.u, v=s.v, d=s.d, e=s.e, flags=np.array([s.box_feasible, s.iterate_bound_ok]),
             obj=np.array([h.objective for h in s.history]), rms=np.array([h.rms for h in s.history]),
             lh=np.array(lp.residual_history), lx=lp.x, ph=np.array(pp.residual_history), px=pp.x,
             mode=np.array(mode))
    print("rank", rank, "mode", mode, flush=True)


if __name__ == "__main__":
    main()
