"""Time the host-input join (tensor_join_vectors path) at cfg2 for several
S chunk counts of the streamed H2D/filter overlap."""
import os, sys, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2312_01476_b200 import device as D, datagen
(L, S), c = datagen.config_vectors(sys.argv[1] if len(sys.argv) > 1 else "cfg2")
Lp, Sp = torch.from_numpy(L).pin_memory(), torch.from_numpy(S).pin_memory()
dev = torch.device("cuda:0")
def step(chunks):
    Ld = Lp.to(dev, non_blocking=True)
    if chunks == 0:
        m = D.join_prepared(D.prepare(Ld), D.prepare(Sp.to(dev, non_blocking=True)), c["theta"])
    else:
        m, _ = D.join_streamed(D.prepare(Ld), Sp, c["theta"], chunks=chunks)
    return m.to_host()
for chunks in (0, 4, 8, 16, 32):
    for _ in range(2): step(chunks)
    ts = []
    for _ in range(5):
        torch.cuda.synchronize(); t0 = time.perf_counter(); step(chunks); ts.append(time.perf_counter() - t0)
    print(f"chunks={chunks}: e2e median {1e3*statistics.median(ts):.2f} ms  min {1e3*min(ts):.2f}", flush=True)
