"""e2e timeline of the one-shot call on c3 (EQUIL_VERBOSE=2 prints the setup
phases without synchronising): development aid."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1602_06621_b200 as eq  # noqa: E402
from paper_1602_06621_b200 import configs  # noqa: E402

inst = configs.config(3)
rp = torch.from_numpy(inst.row_ptr).pin_memory().numpy()
c = torch.from_numpy(inst.col).pin_memory().numpy()
v = torch.from_numpy(inst.val).pin_memory().numpy()
out = tuple(torch.empty(k, dtype=torch.float64).pin_memory().numpy()
            for k in (inst.m, inst.n, inst.m, inst.n))
p = eq.EquilibrationParams(alpha=inst.alpha, beta=inst.beta, iterations=100, seed=0)
for k in range(int(os.environ.get("E2E_REPS", "6"))):
    t0 = time.perf_counter()
    eq.sgd_equilibrate_csr(inst.m, inst.n, rp, c, v, p, out=out)
    print(f"one-shot {1e3 * (time.perf_counter() - t0):.1f} ms", file=sys.stderr, flush=True)
