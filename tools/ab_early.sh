EQUIL_EARLY_LONG=1 timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -m gpu -q -x -k "c3 or config1 or golden or random_shapes or long_slice or boundary" 2>&1 | tail -1
timeout 600 python tools/sell_ab.py 3 EQUIL_EARLY_LONG=0 EQUIL_EARLY_LONG=1 EQUIL_EARLY_LONG=0 EQUIL_EARLY_LONG=1 EQUIL_EARLY_LONG=0 EQUIL_EARLY_LONG=1 2>&1 | tail -6
