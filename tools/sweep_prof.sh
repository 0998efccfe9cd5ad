# per-kernel durations (ncu, serialised) of one SGD iteration with the sweep on
EQUIL_SWEEP=${SWEEP:-1} EQUIL_SWEEP_WIDTH=${WIDTH:-4096} EQUIL_SWEEP_STAGES=${STAGES:-2} timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,smsp__inst_executed.sum --clock-control none \
  -k regex:'sweep_kernel|sell_warp_kernel|sell_long_kernel|sgd_update_rows' -s 6 -c 6 --csv --log-file gpurun_out/sweep_ncu.csv \
  python tools/sell_ab.py 3 EQUIL_SELL=1 > gpurun_out/sweep_ncu.log 2>&1
python - <<'P'
import csv
rows=list(csv.reader(l for l in open('gpurun_out/sweep_ncu.csv') if l.startswith('"')))
h=rows[0]; ki=h.index('Kernel Name'); mi=h.index('Metric Name'); vi=h.index('Metric Value'); ii=h.index('ID')
out={}
for r in rows[1:]:
    out.setdefault((r[ii], r[ki][:60]),{})[r[mi]]=r[vi]
for k,v in out.items(): print(k, v)
P
