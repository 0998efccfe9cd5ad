timeout 300 python tools/ncu_target.py 3 2 1 > gpurun_out/pp_plain.log 2>&1 || exit 1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:sgd_iter_kernel -s 1 -c 1 -o gpurun_out/prof_slots python tools/ncu_target.py 3 2 1 > gpurun_out/pp_ncu.log 2>&1
