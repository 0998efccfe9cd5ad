timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "gpu suite rc=$?"; tail -3 gpurun_out/gputests.log
for i in 1 2 3 4 5; do timeout 600 python -m pytest tests/test_gpu_multiprocess.py tests/test_gpu_parity.py -k "multiprocess or two_processes or host_exchange" -m gpu -q 2>&1 | tail -1; done
