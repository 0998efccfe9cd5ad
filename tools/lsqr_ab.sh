# LSQR pass-variant A/B on c4 (same box): ms per LSQR iteration for EQUIL_PASS_VARIANT values
for pv in "$@"; do
  EQUIL_PASS_VARIANT=${pv%% *} timeout 300 python - <<'PY'
import os, sys, time
sys.path.insert(0, os.getcwd())
import paper_1602_06621_b200 as eq
from paper_1602_06621_b200 import configs
inst = configs.config(4); b = configs.rhs(inst)
M = eq.ExplicitMatrix.from_csr(inst.m, inst.n, inst.row_ptr, inst.col, inst.val)
eq.lsqr(M, b, 3, 0.0)
ts = {}
for k in (10, 60, 10, 60):
    t0 = time.perf_counter(); eq.lsqr(M, b, k, 0.0); ts.setdefault(k, []).append(time.perf_counter() - t0)
print("pv", os.environ["EQUIL_PASS_VARIANT"], f"{(min(ts[60]) - min(ts[10])) / 50 * 1e3:.4f} ms/iter", flush=True)
PY
done
