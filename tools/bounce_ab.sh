set -u
for cfg in "4 4 16" "8 4 16" "8 8 16" "12 8 16" "8 8 32" "16 8 16"; do
  set -- $cfg
  echo "threads $1 slots $2 slotMB $3: $(SJB_BOUNCE_THREADS=$1 SJB_BOUNCE_SLOTS=$2 SJB_BOUNCE_SLOT_MB=$3 timeout 300 python tools/e2e_pageable_probe.py 2>&1 | tail -n 2 | tr '\n' ' ')"
done
nproc
