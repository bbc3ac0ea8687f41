set -u
O=gpurun_out
for ch in 8 16; do cp tools/bin/libsjb200_ch$ch.so paper_2312_01476_b200/libsjb200.so; for th in 0.4 0.8; do timeout 120 python tools/profile_join.py --cfg cfg5 --theta $th --iters 6 > $O/ch_${ch}_${th}.log 2>&1; echo "chains $ch theta $th: $(tail -n 2 $O/ch_${ch}_${th}.log | head -1)"; done; done
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "recheck_placements or medium_instances or nan_and_inf or dense_blocks" 2>&1 | tail -n 1
