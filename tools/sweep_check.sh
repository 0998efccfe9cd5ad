timeout 900 python -m pytest tests/test_gpu_sweep.py -x -q 2>&1 | tail -15
EQUIL_VERBOSE=1 timeout 600 python tools/sell_ab.py 3 EQUIL_SWEEP=0 EQUIL_SWEEP=1 EQUIL_SWEEP=1,EQUIL_SWEEP_WIDTH=5120 EQUIL_SWEEP=1,EQUIL_SWEEP_WIDTH=4608 EQUIL_SWEEP=0 2>&1 | grep -v "^\[equil\] create\|^\[equil\] plan\|^\[equil\] sgd" | tee gpurun_out/ab_sweep.log
