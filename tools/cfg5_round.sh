# cfg5 bench lines (every theta), launch list and the dense-recheck capture -> gpurun_out/
set -u
O=gpurun_out
for th in 0.95 0.8 0.6 0.4; do timeout 600 python bench.py --config cfg5 --theta $th > $O/b5_$th.log 2>&1; tail -n 1 $O/b5_$th.log > $O/b5_$th.json; done
C5="python tools/profile_join.py --cfg cfg5 --theta 0.4 --iters 3"
$C5 > /dev/null 2>&1 && timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r2d_launches_cfg5.csv $C5 > /dev/null 2>&1
$C5 > /dev/null 2>&1 && timeout 300 ncu --set full --clock-control none --import-source on -k "regex:recheck_blocks|group_rows|count_rows|emit_sims" -s 4 -c 4 -o $O/r2d_dense_cfg5 $C5 > /dev/null 2>&1
ls $O | grep -E "b5_|r2d"
