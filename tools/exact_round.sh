# canonical sims on raw bf16 operands (cfg4 exact): -m gpu tests, slice probe in both similarity modes
# and with SJB_WIDE_EXACT=group, the exact-mode launch list
set -u
O=gpurun_out; T=${TAG:-ex}
timeout 1500 python -m pytest tests -m gpu -x -q > $O/${T}_gputest.log 2>&1; echo "pytest rc=$?" >> $O/${T}_gputest.log
timeout 600 python tools/cfg4_probe.py 16000 1000000 3 exact,tensor > $O/${T}_probe.log 2>&1
SJB_WIDE_EXACT=group timeout 600 python tools/cfg4_probe.py 16000 1000000 3 exact > $O/${T}_probe_group.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/${T}_launches_cfg4_exact.csv python tools/cfg4_probe.py 16000 1000000 1 exact > /dev/null 2>&1
tail -n 3 $O/${T}_gputest.log; tail -n 2 $O/${T}_probe.log; tail -n 1 $O/${T}_probe_group.log
