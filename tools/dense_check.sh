timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "gpu suite rc=$?"; tail -3 gpurun_out/gputests.log
for i in 1 2 3; do timeout 120 python tools/c2_probe.py; done
