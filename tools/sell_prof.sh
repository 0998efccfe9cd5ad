# SELL traversal: variant A/B, launch list and one full capture of the SELL kernel
mkdir -p gpurun_out
timeout 600 python tools/sell_ab.py 3 EQUIL_SELL=0 EQUIL_SELL_VARIANT=0 EQUIL_SELL_VARIANT=5 EQUIL_SELL_VARIANT=6 EQUIL_SELL_VARIANT=7 > gpurun_out/sell_ab.log 2>&1
cat gpurun_out/sell_ab.log | tail -5
timeout 300 python tools/ncu_target.py 3 3 1 > gpurun_out/nt.log 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_sell.csv python tools/ncu_target.py 3 3 1 > gpurun_out/ncu_l.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"sgd_sell_kernel|sgd_iter_kernel" -s 2 -c 2 -o gpurun_out/prof_sell python tools/ncu_target.py 3 3 1 > gpurun_out/ncu_f.log 2>&1
tail -2 gpurun_out/ncu_f.log
