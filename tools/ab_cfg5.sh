# A/B of the dense recheck kernels at cfg5 (run on the GPU box)
set -u
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "recheck_placements or medium_instances or nan_and_inf or dense_blocks" > $O/ab_tests.log 2>&1; echo "tests rc=$?" >> $O/ab_tests.log
for th in 0.4 0.8; do
  timeout 120 python tools/profile_join.py --cfg cfg5 --theta $th --iters 6 > $O/ab_blocks_$th.log 2>&1
  SJB_DENSE_RECHECK=rows timeout 120 python tools/profile_join.py --cfg cfg5 --theta $th --iters 6 > $O/ab_rows_$th.log 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ab_launches_cfg5.csv python tools/profile_join.py --cfg cfg5 --theta 0.4 --iters 3 > /dev/null 2>&1
tail -2 $O/ab_tests.log; tail -n 2 $O/ab_*_0.*.log
