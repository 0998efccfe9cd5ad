"""The interleaved slices' stream layouts: every slice 1-wide
(EQUIL_SELL_QUAD=0) and nearly every slice in the quad layout
(EQUIL_QUAD_MIN=4: padding and tails of short rows) must give the same
bit-exact trajectories as the default.  The knobs are read once per process,
so the parity subset runs in a child pytest per layout."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUBSET = ("random_shapes or config1 or lsqr_bit_exact or long_slice_variants or boundary "
          "or operator_path or operator_lsqr")


@pytest.mark.parametrize("env", [{"EQUIL_SELL_QUAD": "0"}, {"EQUIL_QUAD_MIN": "4"}],
                         ids=["one_wide", "quad_everywhere"])
def test_parity_subset_under_layout(env):
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-k", SUBSET,
                        "-p", "no:cacheprovider",
                        "tests/test_gpu_parity.py", "tests/test_gpu_operator.py"],
                       cwd=ROOT, env=dict(os.environ, **env), capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout
