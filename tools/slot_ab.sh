timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for s in 1 0 1 0; do echo "== slots $s"; EQUIL_SLOTS=$s timeout 300 python tools/perf_probe.py 3 2>&1 | tail -1 | cut -c1-260; done
