C5="python tools/profile_join.py --cfg cfg5 --theta 0.4 --iters 3"
$C5 > gpurun_out/p5.log 2>&1 && ncu --set full --clock-control none --import-source on -k "regex:recheck_grouped|segsort_small|group_rows|compact_rows|join_filter" -s 6 -c 5 -o gpurun_out/r2_cfg5_full $C5 > gpurun_out/p5ncu.log 2>&1
tail -3 gpurun_out/p5ncu.log
