free -g | head -2
EQUIL_VERBOSE=1 timeout 1200 python tools/perf_probe.py 5 > gpurun_out/c5.log 2>&1
tail -5 gpurun_out/c5.log | cut -c1-400
nvidia-smi --query-gpu=memory.used,memory.total --format=csv
