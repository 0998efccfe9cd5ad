"""Default mempool high-water marks across repeated one-shot c3 calls (development aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from cuda import cudart
import paper_1602_06621_b200 as eq
from paper_1602_06621_b200 import configs
inst = configs.config(3)
rp = torch.from_numpy(inst.row_ptr).pin_memory().numpy()
c = torch.from_numpy(inst.col).pin_memory().numpy()
v = torch.from_numpy(inst.val).pin_memory().numpy()
out = tuple(torch.empty(k, dtype=torch.float64).pin_memory().numpy() for k in (inst.m, inst.n, inst.m, inst.n))
p = eq.EquilibrationParams(alpha=inst.alpha, beta=inst.beta, iterations=100, seed=0)
err, pool = cudart.cudaDeviceGetDefaultMemPool(0)
def stat():
    r = {}
    for nm, a in (("reserved", cudart.cudaMemPoolAttr.cudaMemPoolAttrReservedMemCurrent), ("reserved_high", cudart.cudaMemPoolAttr.cudaMemPoolAttrReservedMemHigh), ("used_high", cudart.cudaMemPoolAttr.cudaMemPoolAttrUsedMemHigh)):
        e, val = cudart.cudaMemPoolGetAttribute(pool, a)
        r[nm] = round(int(val) / 2**30, 2)
    return r
if os.environ.get("RESIDENT"):
    M = eq.ExplicitMatrix.from_csr(inst.m, inst.n, inst.row_ptr, inst.col, inst.val)
    for _ in range(3):
        eq.sgd_equilibrate(M, p)
    print("resident handle", stat(), flush=True)
    if os.environ.get("RESIDENT") == "closed":
        M.close()
for k in range(int(os.environ.get("E2E_REPS", "12"))):
    t0 = time.perf_counter()
    eq.sgd_equilibrate_csr(inst.m, inst.n, rp, c, v, p, out=out)
    print(f"call {k}: {1e3 * (time.perf_counter() - t0):.1f} ms", stat(), flush=True)
