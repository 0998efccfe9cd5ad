for c in 0 1 2 3 0 1; do echo "== conc $c"; EQUIL_CONC=$c timeout 300 python tools/perf_probe.py 3 2>&1 | tail -1 | cut -c1-200; done
EQUIL_CONC=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "sgd" 2>&1 | tail -2
