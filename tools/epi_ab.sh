set -u
O=gpurun_out
timeout 300 python tools/cfg4_probe.py 16000 1000000 3 tensor,exact > $O/e8.log 2>&1; tail -n 2 $O/e8.log
cp tools/bin/libsjb200_epi16.so paper_2312_01476_b200/libsjb200.so
timeout 300 python tools/cfg4_probe.py 16000 1000000 3 tensor,exact > $O/e16.log 2>&1; tail -n 2 $O/e16.log
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "bf16 or wide" > $O/e16_tests.log 2>&1; tail -n 2 $O/e16_tests.log
