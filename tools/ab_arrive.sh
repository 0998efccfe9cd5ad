timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "long_slice or config1 or lsqr or boundary" 2>&1 | tail -1
for lib in "" lanearr "" lanearr; do
  if [ -n "$lib" ]; then export EQUIL_LIB=$PWD/paper_1602_06621_b200/libequil_b200_$lib.so; else unset EQUIL_LIB; fi
  echo -n "lib=${lib:-warp-arrive} "; timeout 240 python tools/sell_ab.py 3 EQUIL_SELL_LVARIANT=0 2>&1 | tail -1
  bash tools/lsqr_ab.sh 0 | sed "s/^/lib=${lib:-warp-arrive} /"
done
