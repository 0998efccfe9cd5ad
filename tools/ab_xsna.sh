# integration binding + A/B of L1 no-allocate gathers for A's rows (xs)
timeout 600 python -m pytest tests/test_integration.py -m gpu -q 2>&1 | tail -2
for lib in "" xsna1 xsna2 "" xsna1 xsna2; do
  if [ -n "$lib" ]; then export EQUIL_LIB=$PWD/paper_1602_06621_b200/libequil_b200_$lib.so; else unset EQUIL_LIB; fi
  echo -n "lib=${lib:-default} "; timeout 240 python tools/sell_ab.py 3 EQUIL_SELL_LVARIANT=0 2>&1 | tail -1
done
unset EQUIL_LIB
