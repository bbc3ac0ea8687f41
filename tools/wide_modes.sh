# wide-filter time attribution on one GPU (see tools/wide_modes.py): the default
# build's 1-CTA filter, then the A/B build's cta_group::2 filter; each also as an ncu
# launch list of the filter kernels (time + tensor-pipe activity per launch)
set -u
O=gpurun_out; T=${TAG:-wm}; N="${WM_SIZE:-16000 1000000}"
M="gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"
timeout 600 python tools/wide_modes.py $N 3 > $O/${T}_single.log 2>&1
timeout 600 ncu --metrics $M --clock-control none -k regex:filter_kernel --csv --log-file $O/${T}_single_ncu.csv \
  python tools/wide_modes.py $N 1 > /dev/null 2>&1
if [ -n "${WM_AB:-1}" ]; then
  SJB_NVCC_EXTRA=-DSJB_AB_KERNELS=1 python -c "from paper_2312_01476_b200 import build as B; B.build(force=True)"
  VARIANTS=${WM_VARIANTS:-mma2} timeout 600 python tools/wide_modes.py $N 3 > $O/${T}_ab.log 2>&1
  VARIANTS=${WM_VARIANTS:-mma2} timeout 600 ncu --metrics $M --clock-control none -k regex:filter_kernel --csv \
    --log-file $O/${T}_ab_ncu.csv python tools/wide_modes.py $N 1 > /dev/null 2>&1
fi
cat $O/${T}_single.log $O/${T}_ab.log 2>/dev/null | grep mode
