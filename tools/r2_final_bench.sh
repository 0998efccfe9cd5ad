nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gputests.log 2>&1; echo "gpu suite rc=$?"; tail -3 gpurun_out/gputests.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err; echo "ref rc=$?"
