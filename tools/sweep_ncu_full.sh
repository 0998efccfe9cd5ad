# full ncu capture of one sweep_kernel launch + source-level stall samples
EQUIL_SWEEP=1 EQUIL_SWEEP_SERIAL=1 EQUIL_SWEEP_WIDTH=${WIDTH:-4096} EQUIL_SWEEP_STAGES=${STAGES:-2} timeout 900 ncu --set full --import-source on --clock-control none \
  -k regex:'sweep_kernel' -s 3 -c 1 -o gpurun_out/sweep_full -f \
  python tools/sell_ab.py 3 EQUIL_SELL=1 > gpurun_out/sweep_full.log 2>&1
ncu -i gpurun_out/sweep_full.ncu-rep --page source --csv > gpurun_out/sweep_full_source.csv 2>/dev/null
ncu -i gpurun_out/sweep_full.ncu-rep --page raw --csv > gpurun_out/sweep_full_raw.csv 2>/dev/null
ls -la gpurun_out/sweep_full*
