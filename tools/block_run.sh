for mb in 30 50 60 80; do echo "== $mb"; EQUIL_BLOCK_MB=$mb timeout 1200 python tools/perf_probe.py 5 2>&1 | tail -1 | cut -c1-200; done
