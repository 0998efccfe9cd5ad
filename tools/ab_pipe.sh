for t in base p6 p4 p3 base p6; do
  if [ $t = base ]; then L=paper_1602_06621_b200/libequil_b200.so; else L=paper_1602_06621_b200/libequil_b200_$t.so; fi
  for c in 1 3; do
  echo "== $t conc$c"; EQUIL_CONC=$c EQUIL_LIB=$PWD/$L timeout 300 python tools/perf_probe.py 3 2>&1 | tail -1 | cut -c140-200
  done
done
