# A/B build: the two-stage cta_group::2 wide filter (SJB_WIDE_MMA2=2): parity test, then
# the mode attribution beside the 1-CTA kernel, then an ncu launch list of the filters
set -u
O=gpurun_out; T=${TAG:-m2s}; N="${WM_SIZE:-16000 1000000}"
M="gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"
SJB_NVCC_EXTRA=-DSJB_AB_KERNELS=1 python -c "from paper_2312_01476_b200 import build as B; B.build(force=True)"
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "mma2" > $O/${T}_test.log 2>&1; echo "pytest rc=$?" >> $O/${T}_test.log
VARIANTS=${WM_VARIANTS:-mma2s,single} MODES=${WM_MODES:-0,1,2} timeout 600 python tools/wide_modes.py $N 3 > $O/${T}_modes.log 2>&1
VARIANTS=mma2s MODES=0 timeout 600 ncu --metrics $M --clock-control none -k regex:filter_kernel --csv \
  --log-file $O/${T}_ncu.csv python tools/wide_modes.py $N 1 > /dev/null 2>&1
tail -n 3 $O/${T}_test.log; grep mode $O/${T}_modes.log
