"""bench.py's N > 1 path end to end on the one GPU of this project: two ranks
under torch.distributed.run (gloo barriers), the library's POSIX shared-memory
host exchange in place of NCCL (EQUIL_HOST_EXCHANGE=2; NCCL refuses two ranks
on one GPU), real CUDA IPC peer stores (exchange "p2p"), the sharded setup, and
rank 0's check that the sharded c3 run equals one GPU's bit for bit."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_bench_two_ranks_one_gpu():
    env = dict(os.environ, EQUIL_HOST_EXCHANGE="2", EQUIL_SHM_SLOT_MB="64")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
           "--steps", "2", "--warmup", "1", "--e2e-steps", "1", "--no-cpu-baseline",
           "--dist-backend", "gloo", "--device", "0"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert d["exchange"] == "p2p"
    assert d["check"] == {"bit_identical_to_1gpu": True}
    assert d["e2e"]["value"] > 0
