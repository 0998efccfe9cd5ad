"""Matrix creation probe (development aid): c3 from pinned host CSR, twice."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1602_06621_b200 as eq  # noqa: E402
from paper_1602_06621_b200 import configs  # noqa: E402

inst = configs.config(3)
rp = torch.from_numpy(inst.row_ptr).pin_memory().numpy()
c = torch.from_numpy(inst.col).pin_memory().numpy()
v = torch.from_numpy(inst.val).pin_memory().numpy()
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 1):
    M = eq.ExplicitMatrix.from_csr(inst.m, inst.n, rp, c, v)
    M.close()
print("ok")
