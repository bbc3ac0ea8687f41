set -u
O=gpurun_out
for a in 4 8 16; do SJB_AGG_CTAS=$a timeout 120 python tools/profile_join.py --cfg cfg5 --theta 0.4 --iters 6 > $O/agg_$a.log 2>&1; echo "agg $a: $(tail -n 2 $O/agg_$a.log | head -1)"; done
SJB_AGG_CTAS=8 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ab_launches_cfg5.csv python tools/profile_join.py --cfg cfg5 --theta 0.4 --iters 3 > /dev/null 2>&1
