"""The CUDA path on the CHECKED build (libequil_b200_checked.so, built with
-DEQ_CHECKED by paper_1602_06621_b200/build.py).  compute-sanitizer is closed
on this GPU pool, so the kernels carry their own assertions, which trap:

  * every gather of the SGD / LSQR traversals stays inside its vector
    (sell_warp_kernel, sell_long_kernel);
  * the warp-specialised long-slice ring: a stage the chain warp consumes holds
    exactly the round it waits for (stagers tag each stage before arriving on
    its full barrier) -- a hand-off bug in the mbarrier ring trips it;
  * the canonical reduction never writes partials past their buffer (the
    m + n-term history reductions);
  * the transpose's scatter positions stay inside the arrays.

Each workload also compares its results with the oracle (tests/_checked_worker.py)."""
import os
import subprocess
import sys

import pytest

from paper_1602_06621_b200 import build as B

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("case,env", [
    ("c1", {}),
    ("c3s", {}),
    ("c3s", {"EQUIL_BLOCK_MB": "0.1"}),         # column-block rounds and their carries
    ("c3s", {"EQUIL_SPLIT_EPI": "0"}),         # fused epilogue in the traversals
    ("c3s", {"EQUIL_SWEEP": "0"}),             # long rows on the long-slice kernel's ring
    ("c3s", {"EQUIL_SWEEP": "0", "EQUIL_SELL_LVARIANT": "3"}),  # another ring shape (batch 2, 15 stagers)
    ("c3s", {"EQUIL_SWEEP_WIDTH": "700", "EQUIL_SWEEP_STAGES": "3"}),  # narrow sweep panels
])
def test_checked_build_clean(case, env):
    if not os.path.exists(B.CHECKED_LIB):
        pytest.fail("libequil_b200_checked.so missing: run __graft_entry__.build()")
    e = dict(os.environ, EQUIL_LIB=B.CHECKED_LIB, **env)
    r = subprocess.run([sys.executable, os.path.join(HERE, "_checked_worker.py"), case], env=e,
                       capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert "EQ_CHECK failed" not in out, out[-4000:]
    assert r.returncode == 0 and f"ok {case} build_flags 1" in out, out[-4000:]
