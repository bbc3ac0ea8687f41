#!/bin/bash
for th in 0.8 0.4; do
 for m in 0 1; do echo "single mode $m th $th: $(SJB_DEBUG_MODE=$m timeout 120 python tools/profile_join.py --cfg cfg5 --theta $th --iters 3 2>&1 | tail -1)"; done
 echo "pair mode 0 th $th: $(SJB_FILTER=pair timeout 120 python tools/profile_join.py --cfg cfg5 --theta $th --iters 3 2>&1 | tail -1)"
done
