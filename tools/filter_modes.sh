#!/bin/bash
# time the cfg2 join under each diagnostic mode of the filter kernel
for m in ${MODES:-0 1 2}; do
  echo "== mode $m"; SJB_DEBUG_MODE=$m timeout 300 python tools/profile_join.py --iters 3 2>&1 | tail -2
done
