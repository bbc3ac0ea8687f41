# dense-recheck iteration on the GPU box: parity subset, cfg5 timings, block stats, launch list
set -u
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "recheck_placements or medium_instances or nan_and_inf or dense_blocks" > $O/ab_tests.log 2>&1; tail -n 2 $O/ab_tests.log
for th in 0.4 0.6 0.8; do timeout 120 python tools/profile_join.py --cfg cfg5 --theta $th --iters 6 > $O/p_$th.log 2>&1; tail -n 2 $O/p_$th.log; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ab_launches_cfg5.csv python tools/profile_join.py --cfg cfg5 --theta 0.4 --iters 3 > /dev/null 2>&1
cp tools/bin/libsjb200_stats.so paper_2312_01476_b200/libsjb200.so && for th in 0.4 0.8; do timeout 120 python tools/blk_stats.py cfg5 $th 2>&1 | tail -n 1; done
