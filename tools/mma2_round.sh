set -u
O=gpurun_out
SJB_WIDE_MMA2=1 timeout 300 python tools/cfg4_probe.py 16000 1000000 3 tensor > $O/m2_on.log 2>&1; tail -n 1 $O/m2_on.log
SJB_WIDE_MMA2=0 timeout 300 python tools/cfg4_probe.py 16000 1000000 3 tensor > $O/m2_off.log 2>&1; tail -n 1 $O/m2_off.log
SJB_WIDE_MMA2=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/m2_launches.csv python tools/cfg4_probe.py 16000 1000000 1 tensor > /dev/null 2>&1
