#!/bin/bash
# ncu evidence for one round (run on the GPU box; each command first runs
# clean without ncu).  Outputs land in gpurun_out/; tools/ncu_summary.py
# turns them into profiles/<tag>_*.json.
set -u
TAG=${TAG:-r1}
O=gpurun_out
mkdir -p $O
C2="python tools/profile_join.py --iters 2"
C4="python tools/cfg4_probe.py 16000 1000000 1 tensor"
C5="python tools/profile_join.py --cfg cfg5 --theta 0.4 --iters 3"
$C2 > /dev/null && ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/${TAG}_launches_cfg2.csv $C2 > /dev/null 2>&1
$C2 > /dev/null && ncu --set full --clock-control none --import-source on -k regex:join_filter \
  -s 1 -c 1 -o $O/${TAG}_filter_cfg2 $C2 > /dev/null 2>&1
$C4 > /dev/null && ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/${TAG}_launches_cfg4.csv $C4 > /dev/null 2>&1
$C4 > /dev/null && ncu --set full --clock-control none -k "regex:filter_kernel|recheck_pending" -s 2 -c 2 \
  -o $O/${TAG}_wide_cfg4 $C4 > /dev/null 2>&1
$C5 > /dev/null && ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/${TAG}_launches_cfg5.csv $C5 > /dev/null 2>&1
$C5 > /dev/null && ncu --set full --clock-control none --import-source on \
  -k "regex:recheck_blocks|group_rows_agg|count_rows_agg|emit_sims" -s 4 -c 4 \
  -o $O/${TAG}_dense_cfg5 $C5 > /dev/null 2>&1
ls -la $O | grep $TAG
