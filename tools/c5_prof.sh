# c5 (2e7 x 1e6, nnz 1e9) on one GPU: per-kernel times, SELL vs staged, with column blocks
mkdir -p gpurun_out
for sell in 1 0; do
  EQUIL_SELL=$sell timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct --clock-control none --csv --log-file gpurun_out/c5_launches_sell$sell.csv python tools/ncu_target.py 5 2 1 > gpurun_out/c5_ncu_$sell.log 2>&1
  tail -1 gpurun_out/c5_ncu_$sell.log
done
