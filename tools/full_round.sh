# full GPU validation: tests, smoke, cfg5 bench lines
set -u
O=gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gputest.log 2>&1; echo "pytest rc=$?" >> $O/gputest.log
for th in 0.4 0.8; do timeout 600 python bench.py --config cfg5 --theta $th > $O/b5_$th.log 2>&1; tail -n 1 $O/b5_$th.log > $O/b5_$th.json; done
tail -n 2 $O/smoke.log; tail -n 3 $O/gputest.log
