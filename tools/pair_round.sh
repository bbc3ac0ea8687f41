set -u
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "bf16 or wide_pair" > $O/pair_tests.log 2>&1; tail -n 3 $O/pair_tests.log
timeout 300 python tools/cfg4_probe.py 16000 1000000 3 tensor > $O/pair_probe.log 2>&1; tail -n 4 $O/pair_probe.log
SJB_WIDE_PAIR=0 timeout 300 python tools/cfg4_probe.py 16000 1000000 3 tensor > $O/nopair_probe.log 2>&1; tail -n 4 $O/nopair_probe.log
