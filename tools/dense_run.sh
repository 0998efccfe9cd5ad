timeout 900 python -m pytest tests -m gpu -x -q -k "dense or dn or variants" 2>&1 | tail -2
for c in 1 0 1 0; do echo "== conc $c"; EQUIL_CONC=$c timeout 300 python tools/perf_probe.py 2 2>&1 | tail -1 | cut -c1-220; done
