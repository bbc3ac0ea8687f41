"""Block statistics of the cluster-blocked dense recheck (library built with
SJB_NVCC_EXTRA=-DSJB_BLK_STATS=1): python tools/blk_stats.py cfg5 0.4"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2312_01476_b200 import _lib, datagen, device as D

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
theta = float(sys.argv[2]) if len(sys.argv) > 2 else 0.4
(L, S), c = datagen.config_vectors(cfg)
PL, PS = D.prepare(torch.from_numpy(L).cuda()), D.prepare(torch.from_numpy(S).cuda())
lib = _lib.lib()
out = (ctypes.c_int64 * 16)()
for it in range(2):
    lib.sjb_debug_blk_stats(out)
    m = D.join_prepared(PL, PS, theta)
    torch.cuda.synchronize()
    lib.sjb_debug_blk_stats(out)
    v = list(out)
    print(f"{cfg} theta={theta} matches={m.n_matches} cand={m.n_candidates}: blocks dense {v[0]} "
          f"big {v[1]} union-overflow {v[2]} low-density {v[3]}; candidates dense {v[4]} "
          f"sparse {v[5]}; mean dense union {v[6] / max(1, v[0]):.1f}", flush=True)
    names = ["fetch", "rows", "insert", "sort+hidx", "mask", "tma-wait", "compute", "sparse"]
    tot = sum(v[8:16]) or 1
    print("  cycles (CTA thread 0): " + ", ".join(f"{n} {100 * c / tot:.1f}%" for n, c in zip(names, v[8:16])),
          f"total {tot:.3e}", flush=True)
