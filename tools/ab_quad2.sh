# quad layout round 2: LSQR B=4 quad, no param-struct local copies; multiprocess test x3
for i in 1 2 3; do timeout 600 python -m pytest tests/test_gpu_multiprocess.py -m gpu -q 2>&1 | tail -1; done
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "gpu suite rc=$?"; tail -4 gpurun_out/gputests.log
timeout 600 python tools/sell_ab.py 3 EQUIL_SELL_QUAD=1 EQUIL_SELL_QUAD=0 EQUIL_SELL_QUAD=1 EQUIL_SELL_QUAD=0 2>&1 | tail -4
for q in 1 0 1 0; do EQUIL_SELL_QUAD=$q bash tools/lsqr_ab.sh 0 2>&1 | sed "s/^/quad=$q /"; done
