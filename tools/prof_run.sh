python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/b_small.json 2> gpurun_out/b_small.err || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_bench.log 2>&1
timeout 300 python tools/ncu_target.py 3 3 1 > gpurun_out/pp_plain.log 2>&1 || exit 1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:sgd_iter_kernel -s 2 -c 2 -o gpurun_out/prof_r1b python tools/ncu_target.py 3 3 1 > gpurun_out/pp_ncu.log 2>&1
