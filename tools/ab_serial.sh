# concurrent vs per-matrix traversal order (separate processes: the knob is read once)
for v in 0 3 4 0 3 4; do EQUIL_SERIAL=$v timeout 240 python tools/sell_ab.py 3 EQUIL_SELL_VARIANT=0 2>&1 | tail -1 | sed "s/^/serial=$v /"; done
EQUIL_SERIAL=3 timeout 300 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x 2>&1 | tail -1
