# round-2 (column sweep) evidence: GPU suite, bench (ours + reference arm), bench
# launch list, one full capture of the SGD iteration kernels (sweep, warp slices,
# update), source-level stall samples of the sweep kernel, LSQR launch list
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gputests.log 2>&1; echo "gpu suite rc=$?"; tail -3 gpurun_out/gputests.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -c 600 gpurun_out/bench.json
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err; echo "ref rc=$?"
timeout 300 python tools/ncu_target.py 3 3 1 > gpurun_out/nt.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-extras > gpurun_out/ncu_bench.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"sweep_kernel|sell_warp|sell_long|sgd_update" -s 6 -c 3 -f -o gpurun_out/prof_r2g_sgd python tools/ncu_target.py 3 3 1 > gpurun_out/ncu_f.log 2>&1; echo "ncu full rc=$?"; tail -2 gpurun_out/ncu_f.log
timeout 300 python tools/lsqr_prof.py 10 > gpurun_out/lp.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_lsqr.csv python tools/lsqr_prof.py 10 > gpurun_out/lp_ncu.log 2>&1; echo "ncu lsqr rc=$?"
bash tools/sweep_ncu_full.sh
