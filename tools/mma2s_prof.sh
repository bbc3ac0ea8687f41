# A/B build: two-stage cta_group::2 wide filter: modes 0/1/3, then one ncu --set full capture
set -u
O=gpurun_out; T=${TAG:-m2p}; N="${WM_SIZE:-16000 1000000}"
SJB_NVCC_EXTRA=-DSJB_AB_KERNELS=1 python -c "from paper_2312_01476_b200 import build as B; B.build(force=True)"
VARIANTS=mma2s MODES=${WM_MODES:-0,1,3} timeout 600 python tools/wide_modes.py $N 3 > $O/${T}_modes.log 2>&1
VARIANTS=mma2s MODES=0 timeout 900 ncu --set full --import-source on --clock-control none -k regex:filter_kernel \
  --launch-skip 1 --launch-count 1 -o $O/${T}_full -f python tools/wide_modes.py $N 1 > $O/${T}_ncu.log 2>&1
grep mode $O/${T}_modes.log
