timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
EQUIL_VERBOSE=1 timeout 600 python tools/e2e_probe.py > gpurun_out/e2e_probe.log 2>&1
timeout 300 python tools/perf_probe.py 3 2>&1 | tail -1 | cut -c1-200
