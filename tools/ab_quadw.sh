# quad layout with 256-bit value loads: layout parity, then c3 / c4 A/B
timeout 900 python -m pytest tests/test_gpu_layouts.py -m gpu -x -q 2>&1 | tail -1
for qm in 513 64 32 513 64 32; do EQUIL_QUAD_MIN=$qm timeout 240 python tools/sell_ab.py 3 EQUIL_SELL_VARIANT=0 2>&1 | tail -1 | sed "s/^/qmin=$qm /"; done
for qm in 513 64 513 64; do EQUIL_QUAD_MIN=$qm bash tools/lsqr_ab.sh 0 2>&1 | sed "s/^/qmin=$qm /"; done
