# ncu --set full + source of the prep kernels (cfg2 S normalise, cfg3 subword
# gather) -- run clean first
set -u
O=gpurun_out
python tools/prep_profile.py > /dev/null && ncu --set full --clock-control none --import-source on \
  -k "regex:normalize_pipe|subword_gather" -s 2 -c 2 -o $O/prep_full python tools/prep_profile.py > $O/prep_ncu.log 2>&1
tail -n 2 $O/prep_ncu.log
timeout 120 python tools/prep_bench.py > $O/prep_bench.json 2>&1; tail -n 30 $O/prep_bench.json
