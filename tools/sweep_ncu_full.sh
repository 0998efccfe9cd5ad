# full ncu capture of one sweep_kernel launch + source-level stall samples
timeout 900 ncu --set full --import-source on --clock-control none \
  -k regex:'sweep_kernel' -s 1 -c 1 -o gpurun_out/sweep_full -f \
  python tools/ncu_target.py 3 3 1 > gpurun_out/sweep_full.log 2>&1
ncu -i gpurun_out/sweep_full.ncu-rep --page source --csv > gpurun_out/sweep_full_source.csv 2>/dev/null
ls -la gpurun_out/sweep_full*
