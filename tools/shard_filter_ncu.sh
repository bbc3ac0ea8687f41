# the pair filter at a full cfg4 rank share (125k x 4M) under ncu: time, clock, tensor-pipe activity, DRAM / L2
set -u
O=gpurun_out; T=${TAG:-sf}
M="gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_lookup_hit.sum,lts__t_sectors_srcunit_tex_lookup_miss.sum,smsp__issue_active.avg.pct_of_peak_sustained_active"
timeout 1500 ncu --metrics $M --clock-control none -k regex:filter_kernel --csv --log-file $O/${T}_filter.csv \
  python tools/cfg4_probe.py ${SF_SIZE:-125000 4000000} 1 tensor > $O/${T}_probe.log 2>&1
tail -n 1 $O/${T}_probe.log
python - <<PY
import csv
rows=[r for r in csv.reader(open("gpurun_out/${T}_filter.csv")) if len(r)>10]
h=rows[0]; ii=h.index("ID"); mi=h.index("Metric Name"); vi=h.index("Metric Value")
d={}
for r in rows[1:]: d.setdefault(r[ii],{})[r[mi].split(".")[0]+"."+r[mi].split(".")[1]]=r[vi]
for k,v in d.items(): print(k, v)
PY
