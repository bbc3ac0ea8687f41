"""Per-rank device work of the strong-scaling bench on one GPU: rank 0's R
shard of |R|/N rows against all of S (prepare both + join, as each rank does
after the S broadcast), for N = 1, 2, 4, 8.  The broadcast itself (NCCL over
NVLink) is not measured here; the ratio (step at N=1) / (N * step at N)
bounds the strong-scaling efficiency from the per-rank compute side."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2312_01476_b200 import datagen, device as D
from paper_2312_01476_b200 import multigpu as MG

(L, S), c = datagen.config_vectors("cfg2")
dev = torch.device("cuda", 0)
Ld, Sd = torch.from_numpy(L).to(dev), torch.from_numpy(S).to(dev)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
base = None
for world in (1, 2, 4, 8):
    r0, r1 = MG.shard_range(L.shape[0], 0, world)
    R = Ld[r0:r1]
    for _ in range(3):
        D.join_prepared(D.prepare(R), D.prepare(Sd), c["theta"], left_base=r0)
    ts = []
    for _ in range(10):
        torch.cuda.synchronize()
        ev[0].record()
        D.join_prepared(D.prepare(R), D.prepare(Sd), c["theta"], left_base=r0)
        ev[1].record()
        torch.cuda.synchronize()
        ts.append(ev[0].elapsed_time(ev[1]))
    t = statistics.median(ts)
    base = base or t
    print(f"N={world}: rank-0 shard {r1 - r0} x {S.shape[0]}: {t:.2f} ms per step; "
          f"compute-side efficiency {base / (world * t):.3f}", flush=True)
