set -u
O=gpurun_out
for a in 8 16; do SJB_AGG_CTAS=$a timeout 120 python tools/profile_join.py --cfg cfg5 --theta 0.4 --iters 6 > $O/agg_$a.log 2>&1; echo "agg256 $a: $(tail -n 2 $O/agg_$a.log | head -1)"; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ab_launches_cfg5.csv python tools/profile_join.py --cfg cfg5 --theta 0.4 --iters 3 > /dev/null 2>&1
cp tools/bin/libsjb200_agg512.so paper_2312_01476_b200/libsjb200.so
for a in 4 8; do SJB_AGG_CTAS=$a timeout 120 python tools/profile_join.py --cfg cfg5 --theta 0.4 --iters 6 > $O/agg5_$a.log 2>&1; echo "agg512 $a: $(tail -n 2 $O/agg5_$a.log | head -1)"; done
SJB_AGG_CTAS=4 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ab_launches_cfg5b.csv python tools/profile_join.py --cfg cfg5 --theta 0.4 --iters 3 > /dev/null 2>&1
