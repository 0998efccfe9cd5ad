timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1
tail -3 gpurun_out/gputests.log
bash tools/lsqr_ab.sh 0 > gpurun_out/lsqr_ab.log 2>&1
cat gpurun_out/lsqr_ab.log
