import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "ref_golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); run with -m gpu")


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(GOLDEN))


@pytest.fixture(scope="session")
def C():
    import oracle
    return oracle.c_oracle()


def csr_from_golden(g, key):
    import oracle
    if f"{key}_dense" in g:
        d = g[f"{key}_dense"]
        return oracle.CsrArrays(d.shape[0], d.shape[1], dense=d)
    m, n = (int(x) for x in g[f"{key}_shape"])
    return oracle.CsrArrays(m, n, g[f"{key}_rp"], g[f"{key}_col"], g[f"{key}_val"])
