set -u
O=gpurun_out; T=${TAG:-pd}
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "pending or bf16 or mma2 or wide or tensor" > $O/${T}_test.log 2>&1; echo "pytest rc=$?" >> $O/${T}_test.log
SJB_PENDING=gather timeout 600 python tools/cfg4_probe.py 16000 1000000 3 tensor > $O/${T}_gather.log 2>&1
timeout 600 python tools/cfg4_probe.py 16000 1000000 3 tensor > $O/${T}_staged.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/${T}_launches_cfg4.csv python tools/cfg4_probe.py 16000 1000000 1 tensor > /dev/null 2>&1
tail -n 3 $O/${T}_test.log; tail -n 1 $O/${T}_gather.log; tail -n 1 $O/${T}_staged.log
grep -E "recheck_pending|segsort_big" $O/${T}_launches_cfg4.csv | cut -d, -f5,15- | tail -n 4
