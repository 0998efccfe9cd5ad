for v in 0 1 2 0 1 2; do EQUIL_UPD_VARIANT=$v timeout 240 python tools/sell_ab.py 3 EQUIL_SELL_VARIANT=0 2>&1 | tail -1 | sed "s/^/upd=$v /"; done
EQUIL_UPD_VARIANT=2 timeout 300 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -m gpu -q -x -k "c3 or config1 or golden" 2>&1 | tail -1
