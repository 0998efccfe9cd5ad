"""The sharded engine across PROCESSES on one GPU, with the real CUDA IPC path.

Two ranks run as separate processes (tests/_mp_worker.py).  They exchange over a
POSIX shared-memory host transport with a host barrier per exchange
(EQUIL_HOST_EXCHANGE=2; NCCL refuses two ranks on one GPU), and the fused
all-gather maps each peer's gathered-vector buffer with cudaIpcGetMemHandle /
cudaIpcOpenMemHandle, so every SGD epilogue stores its next values into the
other process's buffer -- the code path NVLink peers take, minus the device
barrier (no kernel here ever waits on another rank's kernel).  Every rank must
return the single-GPU result bit for bit: u, v, d, e, flags, the history, and
plain and preconditioned LSQR (src/equilibrate.cpp:138-221, src/lsqr.cpp:85-138).
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_1602_06621_b200 as eq
from paper_1602_06621_b200 import configs

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("p2p", ["1", "0"])
def test_two_processes_bit_identical_to_one_gpu(tmp_path, p2p):
    world = 2
    nid = os.urandom(128).hex()
    env = dict(os.environ, EQUIL_HOST_EXCHANGE="2", EQUIL_P2P=p2p)
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "_mp_worker.py"), str(r),
                               str(world), nid, str(tmp_path / f"r{r}.npz")], env=env,
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
             for r in range(world)]
    logs = []
    for pr in procs:
        try:
            out, _ = pr.communicate(timeout=600)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
        logs.append(out)
        assert pr.returncode == 0, out
    inst = configs.config(3, scale=0.02)
    b = np.random.default_rng(4).standard_normal(inst.m)
    M1 = eq.ExplicitMatrix.from_csr(inst.m, inst.n, inst.row_ptr, inst.col, inst.val)
    ref = eq.sgd_equilibrate(M1, eq.EquilibrationParams(iterations=20, seed=5),
                             eq.DiagnosticsConfig(stride=5))
    rl = eq.lsqr(M1, b, 12, 0.0)
    rp = eq.lsqr_preconditioned(M1, b, eq.EquilibrationParams(iterations=8, seed=2), 12, 0.0)
    for r in range(world):
        got = np.load(tmp_path / f"r{r}.npz")
        assert str(got["mode"]) == ("p2p" if p2p == "1" else "allgather"), logs[r]
        for k in "uvde":
            assert np.array_equal(got[k], getattr(ref, k)), (r, k)
        assert list(got["flags"]) == [ref.box_feasible, ref.iterate_bound_ok]
        assert list(got["obj"]) == [h.objective for h in ref.history]
        assert list(got["rms"]) == [h.rms for h in ref.history]
        assert np.array_equal(got["lh"], rl.residual_history)
        assert np.array_equal(got["lx"], rl.x)
        assert np.array_equal(got["ph"], rp.residual_history)
        assert np.array_equal(got["px"], rp.x)
