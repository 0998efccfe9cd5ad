timeout 300 python tools/lsqr_prof.py 10 > gpurun_out/lp.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_lsqr.csv python tools/lsqr_prof.py 10 > gpurun_out/lp_ncu.log 2>&1
