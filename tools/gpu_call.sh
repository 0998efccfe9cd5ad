timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1
tail -2 gpurun_out/gputests.log
for w in 1 0 1 0; do EQUIL_L2WIN=$w timeout 120 python tools/c2_probe.py; done
