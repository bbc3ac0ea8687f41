# round-end evidence on one GPU: tests, smoke, every bench line, the reference arm, launch lists
set -u
O=gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gputest.log 2>&1; echo "pytest rc=$?" >> $O/gputest.log
timeout 900 python bench.py > $O/fb_cfg2.log 2>&1; tail -n 1 $O/fb_cfg2.log > $O/fb_cfg2.json
timeout 900 python bench.py --config cfg3 > $O/fb_cfg3.log 2>&1; tail -n 1 $O/fb_cfg3.log > $O/fb_cfg3.json
for th in 0.95 0.8 0.6 0.4; do timeout 600 python bench.py --config cfg5 --theta $th > $O/fb_cfg5_$th.log 2>&1; tail -n 1 $O/fb_cfg5_$th.log > $O/fb_cfg5_$th.json; done
tail -n 2 $O/smoke.log; tail -n 3 $O/gputest.log
