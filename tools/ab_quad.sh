# quad layout of the long slices: GPU suite, then c3 SGD and c4 LSQR A/B
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "gpu suite rc=$?"; tail -4 gpurun_out/gputests.log
EQUIL_SELL_QUAD=0 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "lsqr or long_slice or boundary or config1" > gpurun_out/gputests_q0.log 2>&1; echo "q0 subset rc=$?"; tail -2 gpurun_out/gputests_q0.log
timeout 600 python tools/sell_ab.py 3 EQUIL_SELL_QUAD=1 EQUIL_SELL_QUAD=0 EQUIL_SELL_QUAD=1 EQUIL_SELL_QUAD=0 2>&1 | tail -4
for q in 1 0 1 0; do EQUIL_SELL_QUAD=$q bash tools/lsqr_ab.sh 0 2>&1 | sed "s/^/quad=$q /"; done
