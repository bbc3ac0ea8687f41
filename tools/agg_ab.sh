set -u
O=gpurun_out
for v in base per16; do
  if [ $v = per16 ]; then cp tools/bin/libsjb200_per16.so paper_2312_01476_b200/libsjb200.so; fi
  for a in 8 16; do SJB_AGG_CTAS=$a timeout 120 python tools/profile_join.py --cfg cfg5 --theta 0.4 --iters 6 > $O/agg_${v}_$a.log 2>&1; echo "$v ctas $a: $(tail -n 2 $O/agg_${v}_$a.log | head -1)"; done
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ab_launches_cfg5.csv python tools/profile_join.py --cfg cfg5 --theta 0.4 --iters 3 > /dev/null 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "random_shapes or dense_blocks" 2>&1 | tail -n 1
