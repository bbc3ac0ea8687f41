# canonical sims on raw bf16 operands (cfg4 exact): tests of the wide paths, the slice probe with the default
# and with SJB_WIDE_EXACT=rows, and the rows path's launch list
set -u
O=gpurun_out; T=${TAG:-ex}
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q -k "wide or bf16 or cfg4" > $O/${T}_test.log 2>&1; echo "pytest rc=$?" >> $O/${T}_test.log
SJB_WIDE_EXACT=rows timeout 600 python tools/cfg4_probe.py 16000 1000000 3 exact > $O/${T}_probe_rows.log 2>&1
timeout 600 python tools/cfg4_probe.py 16000 1000000 3 exact > $O/${T}_probe_group.log 2>&1
SJB_WIDE_EXACT=rows timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/${T}_launches_cfg4_rows.csv python tools/cfg4_probe.py 16000 1000000 1 exact > /dev/null 2>&1
tail -n 3 $O/${T}_test.log; tail -n 1 $O/${T}_probe_rows.log; tail -n 1 $O/${T}_probe_group.log
grep -E "recheck_segments|filter_kernel|scatter|segsort_big" $O/${T}_launches_cfg4_rows.csv | awk -F'","' '{print substr($5,1,44), $NF}' | tail -n 4
