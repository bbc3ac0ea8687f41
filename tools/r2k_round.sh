# final cfg4 evidence after the sort changes (TAG names the outputs): smoke, -m gpu tests, default bench,
# cfg4 bench lines in both similarity modes, slice launch lists in both modes, full capture of the pair filter
set -u
O=gpurun_out; T=${TAG:-r2k}
python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> $O/${T}_smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > $O/${T}_gputest.log 2>&1; echo "pytest rc=$?" >> $O/${T}_gputest.log
timeout 900 python bench.py > $O/${T}_bench_cfg2.log 2>&1; tail -n 1 $O/${T}_bench_cfg2.log > $O/${T}_bench_cfg2.json
timeout 1500 python bench.py --config cfg4 --sims tensor > $O/${T}_bench_cfg4_tensor.log 2>&1; tail -n 1 $O/${T}_bench_cfg4_tensor.log > $O/${T}_bench_cfg4_tensor.json
timeout 1500 python bench.py --config cfg4 > $O/${T}_bench_cfg4_exact.log 2>&1; tail -n 1 $O/${T}_bench_cfg4_exact.log > $O/${T}_bench_cfg4_exact.json
for m in tensor exact; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/${T}_launches_cfg4_$m.csv python tools/cfg4_probe.py 16000 1000000 1 $m > /dev/null 2>&1
done
timeout 900 ncu --set full --clock-control none -k "regex:filter_kernel|recheck_pending|segsort_big" -s 3 -c 3 -f \
  -o $O/${T}_wide_cfg4 python tools/cfg4_probe.py 16000 1000000 1 tensor > /dev/null 2>&1
tail -n 2 $O/${T}_smoke.log; tail -n 3 $O/${T}_gputest.log
