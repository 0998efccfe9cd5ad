for t in base pf1 pf2 pf4 sb8 sb6 pf2sb8 base pf2; do
  if [ $t = base ]; then L=paper_1602_06621_b200/libequil_b200.so; else L=paper_1602_06621_b200/libequil_b200_$t.so; fi
  echo "== $t"; EQUIL_LIB=$PWD/$L timeout 300 python tools/perf_probe.py 3 2>&1 | tail -1 | cut -c1-200
done
