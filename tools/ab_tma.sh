# long-slice TMA/cp.async kernel: parity with the variant forced, then c3 A/B
EQUIL_SELL_LVARIANT=10 EQUIL_PASS_VARIANT=10 timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_v10.log 2>&1; tail -3 gpurun_out/gputests_v10.log
timeout 900 python tools/sell_ab.py 3 EQUIL_SELL_LVARIANT=0 EQUIL_SELL_LVARIANT=10 EQUIL_SELL_LVARIANT=11 EQUIL_SELL_LVARIANT=12 EQUIL_SELL_LVARIANT=13 EQUIL_SELL_LVARIANT=14 EQUIL_SELL_LVARIANT=15 \
  EQUIL_SELL_LVARIANT=11,EQUIL_CARVE_LONG=22 EQUIL_SELL_LVARIANT=11,EQUIL_CARVE_LONG=75 EQUIL_SELL_LVARIANT=11,EQUIL_CARVE_LONG=100 EQUIL_SELL_LVARIANT=11,EQUIL_CARVE_LONG=-1 EQUIL_SELL_LVARIANT=0 2>&1 | tee gpurun_out/ab_tma.log
bash tools/lsqr_ab.sh 0 10 11 12 0 2>&1 | tee gpurun_out/ab_tma_lsqr.log
