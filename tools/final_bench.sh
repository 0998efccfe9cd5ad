# bench (ours + reference arm) and the sweep kernel's source-level capture
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err; echo "ref rc=$?"
bash tools/sweep_ncu_full.sh
