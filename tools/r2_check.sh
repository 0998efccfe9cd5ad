# GPU suite + LSQR timing after the sharded setup / slotted LSQR changes
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "gpu suite rc=$?"; tail -15 gpurun_out/gputests.log
bash tools/lsqr_ab.sh 0 2>&1 | tee gpurun_out/lsqr_slot.log
