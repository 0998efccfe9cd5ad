# long-slice TMA/cp.async kernel (3 warps): quick parity, full suites, c3 A/B per spec
EQUIL_SELL_LVARIANT=10 EQUIL_PASS_VARIANT=10 timeout 180 python -m pytest tests/test_gpu_parity.py -q -x -k "random_shapes or config1" > gpurun_out/t_v10_quick.log 2>&1
rc=$?; echo "quick v10 rc=$rc"; tail -2 gpurun_out/t_v10_quick.log
if [ $rc -ne 0 ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -k "not long_slice_variants" > gpurun_out/gputests.log 2>&1; echo "gpu suite rc=$?"; tail -3 gpurun_out/gputests.log
  exit 0
fi
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gputests.log 2>&1; echo "gpu suite rc=$?"; tail -5 gpurun_out/gputests.log
EQUIL_SELL_LVARIANT=10 EQUIL_PASS_VARIANT=10 timeout 900 python -m pytest tests -m gpu -x -q -k "not long_slice_variants" > gpurun_out/gputests_v10.log 2>&1; echo "v10 suite rc=$?"; tail -3 gpurun_out/gputests_v10.log
for spec in EQUIL_SELL_LVARIANT=0 EQUIL_SELL_LVARIANT=10 EQUIL_SELL_LVARIANT=11 EQUIL_SELL_LVARIANT=12 EQUIL_SELL_LVARIANT=13 EQUIL_SELL_LVARIANT=14 EQUIL_SELL_LVARIANT=15 \
  EQUIL_SELL_LVARIANT=11,EQUIL_CARVE_LONG=22 EQUIL_SELL_LVARIANT=11,EQUIL_CARVE_LONG=75 EQUIL_SELL_LVARIANT=11,EQUIL_CARVE_LONG=100 EQUIL_SELL_LVARIANT=11,EQUIL_CARVE_LONG=-1 EQUIL_SELL_LVARIANT=0; do
  timeout 240 python tools/sell_ab.py 3 $spec 2>&1 | tail -1 | tee -a gpurun_out/ab_tma.log
done
bash tools/lsqr_ab.sh 0 10 11 12 0 2>&1 | tee gpurun_out/ab_tma_lsqr.log
