# A/B build of the two-stage cta_group::2 wide filter with 8 and 16 epilogue warps:
# parity test, then the modes; finally an ncu launch list of the last variant's filter
set -u
O=gpurun_out; T=${TAG:-m2e}; N="${WM_SIZE:-16000 1000000}"
M="gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"
for E in ${EPIS:-8 16}; do
  SJB_NVCC_EXTRA="-DSJB_AB_KERNELS=1 -DSJB_WIDE2_EPI=$E" python -c "from paper_2312_01476_b200 import build as B; B.build(force=True)"
  timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "mma2" > $O/${T}_test$E.log 2>&1; echo "pytest rc=$?" >> $O/${T}_test$E.log
  VARIANTS=mma2s MODES=${WM_MODES:-0,1,3} timeout 600 python tools/wide_modes.py $N 3 > $O/${T}_modes$E.log 2>&1
  VARIANTS=mma2s MODES=0 timeout 600 ncu --metrics $M --clock-control none -k regex:filter_kernel --csv \
    --log-file $O/${T}_ncu$E.csv python tools/wide_modes.py $N 1 > /dev/null 2>&1
  echo "EPI=$E"; tail -n 2 $O/${T}_test$E.log; grep mode $O/${T}_modes$E.log; grep filter_kernel $O/${T}_ncu$E.csv | tail -n 2 | cut -d, -f5,13-
done
