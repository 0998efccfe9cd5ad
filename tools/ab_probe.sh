set -x
for t in base w1k w16k lc32 lc32b8 sb2 th1k base; do
  if [ $t = base ]; then L=paper_1602_06621_b200/libequil_b200.so; else L=paper_1602_06621_b200/libequil_b200_$t.so; fi
  echo "== $t"; EQUIL_LIB=$PWD/$L timeout 300 python tools/perf_probe.py 3 2>&1 | tail -1
done
EQUIL_LIB=$PWD/paper_1602_06621_b200/libequil_b200_lc32.so timeout 600 python -m pytest tests -m gpu -x -q -k "sgd" 2>&1 | tail -3
