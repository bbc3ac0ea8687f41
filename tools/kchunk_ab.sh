set -u
O=gpurun_out
timeout 300 python tools/cfg4_probe.py 16000 1000000 3 tensor,exact > $O/k64.log 2>&1; tail -n 2 $O/k64.log
cp tools/bin/libsjb200_k32.so paper_2312_01476_b200/libsjb200.so
timeout 300 python tools/cfg4_probe.py 16000 1000000 3 tensor,exact > $O/k32.log 2>&1; tail -n 2 $O/k32.log
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "bf16 or wide" > $O/k32_tests.log 2>&1; tail -n 2 $O/k32_tests.log
