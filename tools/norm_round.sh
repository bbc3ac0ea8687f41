set -u
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "normalize or rounding_error or streamed or sharded or owner or subword or per_row_band or golden" > $O/norm_tests.log 2>&1; tail -n 2 $O/norm_tests.log
timeout 120 python tools/prep_bench.py > $O/prep_bench.log 2>&1; grep -A4 normalize_cast_cfg2 $O/prep_bench.log | grep '"ms"'
SJB_PREP_HALF=0 timeout 120 python tools/prep_bench.py > $O/prep_bench2.log 2>&1; grep -A4 normalize_cast_cfg2 $O/prep_bench2.log | grep '"ms"'
