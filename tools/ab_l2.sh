for t in base l2h1 l2h2 l2h3 base l2h1 l2h3; do
  if [ $t = base ]; then L=paper_1602_06621_b200/libequil_b200.so; else L=paper_1602_06621_b200/libequil_b200_$t.so; fi
  echo "== $t"; EQUIL_LIB=$PWD/$L timeout 300 python tools/perf_probe.py 3 2>&1 | tail -1 | cut -c1-200
done
