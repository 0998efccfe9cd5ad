set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 300 python tools/perf_probe.py 3 2>&1 | tail -1 | cut -c1-250
EQUIL_BANDS_PER_SM=1 timeout 300 python tools/perf_probe.py 3 2>&1 | tail -1 | cut -c1-250
timeout 300 python tools/ncu_target.py 3 2 1 > gpurun_out/pp_plain.log 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:sgd_panel -s 1 -c 1 -o gpurun_out/prof_panel3 python tools/ncu_target.py 3 2 1 > gpurun_out/pp_ncu.log 2>&1
