set -u
O=gpurun_out; T=${TAG:-srt}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q -k "wide or bf16 or all_pairs or cfg4 or canonical or sort or theta" > $O/${T}_test.log 2>&1; echo "pytest rc=$?" >> $O/${T}_test.log
timeout 600 python tools/cfg4_probe.py 16000 1000000 3 tensor > $O/${T}_cfg4.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:segsort \
  --log-file $O/${T}_launches.csv python tools/cfg4_probe.py 16000 1000000 1 tensor > /dev/null 2>&1
[ -n "${FULL:-}" ] && timeout 600 ncu --set full --import-source on --clock-control none -k regex:segsort_big -s 2 -c 1 -f -o $O/${T}_segsort \
  python tools/cfg4_probe.py 16000 1000000 1 tensor > /dev/null 2>&1
tail -n 2 $O/${T}_test.log; tail -n 1 $O/${T}_cfg4.log; grep segsort_big $O/${T}_launches.csv | awk -F'","' '{print $NF}'
