# cfg4 (wide, raw bf16) check of the current default build: -m gpu tests, the slice probe in
# both similarity modes, the bench line of one rank's share, and the tensor-sims launch list
set -u
O=gpurun_out; T=${TAG:-c4}
if [ -z "${SKIP_TESTS:-}" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $O/${T}_gputest.log 2>&1; echo "pytest rc=$?" >> $O/${T}_gputest.log
fi
C4="python tools/cfg4_probe.py 16000 1000000 3 tensor,exact"
timeout 600 $C4 > $O/${T}_cfg4.log 2>&1
C4="python tools/cfg4_probe.py 16000 1000000 1 tensor"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/${T}_launches_cfg4.csv $C4 > /dev/null 2>&1
if [ -n "${BENCH4:-}" ]; then
  timeout 1200 python bench.py --config cfg4 --sims tensor > $O/${T}_bench_cfg4_tensor.log 2>&1; tail -n 1 $O/${T}_bench_cfg4_tensor.log > $O/${T}_bench_cfg4_tensor.json
fi
tail -n 3 $O/${T}_gputest.log 2>/dev/null; tail -n 3 $O/${T}_cfg4.log
