# GPU tests, bench, launch list and one full capture of the SGD kernels (SELL traversal)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; tail -2 gpurun_out/gputests.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 300 python tools/ncu_target.py 3 3 1 > gpurun_out/nt.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"sell_warp|sell_long|sgd_update" -s 3 -c 3 -o gpurun_out/prof_sell2 python tools/ncu_target.py 3 3 1 > gpurun_out/ncu_f.log 2>&1
tail -2 gpurun_out/ncu_f.log
