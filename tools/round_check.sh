# quick check of the current code on one GPU: smoke, -m gpu tests, the default bench line,
# the per-rank shard probe and the cfg4 slice probe (TAG names the outputs)
set -u
O=gpurun_out; T=${TAG:-chk}
python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> $O/${T}_smoke.log
if [ -z "${SKIP_TESTS:-}" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $O/${T}_gputest.log 2>&1; echo "pytest rc=$?" >> $O/${T}_gputest.log
fi
timeout 900 python bench.py > $O/${T}_cfg2.log 2>&1; tail -n 1 $O/${T}_cfg2.log > $O/${T}_cfg2.json
timeout 600 python tools/shard_probe.py > $O/${T}_shard.log 2>&1
timeout 600 python tools/cfg4_probe.py 16000 1000000 3 tensor,exact > $O/${T}_cfg4.log 2>&1
tail -n 2 $O/${T}_smoke.log; tail -n 3 $O/${T}_gputest.log 2>/dev/null; cat $O/${T}_shard.log | tail -6; cat $O/${T}_cfg4.log | tail -3
