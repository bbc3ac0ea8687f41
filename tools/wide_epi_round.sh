# A/B: the 1-CTA wide filter (canonical sims / fp32 path) with 16 epilogue warps on 32-column chunks
set -u
O=gpurun_out; T=${TAG:-we}
for E in ${EPIS:-16 8}; do
  SJB_NVCC_EXTRA="-DSJB_WIDE_EPI=$E" python -c "from paper_2312_01476_b200 import build as B; B.build(force=True)"
  timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q -k "wide or bf16 or cfg4" > $O/${T}_test$E.log 2>&1; echo "pytest rc=$?" >> $O/${T}_test$E.log
  timeout 600 python tools/cfg4_probe.py 16000 1000000 3 exact,fp32 > $O/${T}_probe$E.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k "regex:filter_kernel|recheck_group" \
    --log-file $O/${T}_launches$E.csv python tools/cfg4_probe.py 16000 1000000 1 exact > /dev/null 2>&1
  echo "EPI=$E"; tail -n 2 $O/${T}_test$E.log; tail -n 2 $O/${T}_probe$E.log; grep -E "filter_kernel|recheck_group" $O/${T}_launches$E.csv | awk -F'","' '{print substr($5,1,36), $NF}' | tail -n 2
done
