timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python tools/lsqr_probe.py 2>&1 | tail -12
timeout 300 python tools/perf_probe.py 3 2>&1 | tail -1 | cut -c1-200
