set -u
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "recheck_placements or medium_instances or nan_and_inf or dense_blocks or random_shapes or golden" 2>&1 | tail -n 2
for v in 1 0; do for th in 0.4 0.8; do SJB_ITEM_GROUPING=$v timeout 120 python tools/profile_join.py --cfg cfg5 --theta $th --iters 6 > $O/it_${v}_$th.log 2>&1; echo "items $v theta $th: $(tail -n 2 $O/it_${v}_$th.log | head -1)"; done; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ab_launches_cfg5.csv python tools/profile_join.py --cfg cfg5 --theta 0.4 --iters 3 > /dev/null 2>&1
