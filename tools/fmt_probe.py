"""Matches-file formatting at cfg2 scale: the GPU writer (layout + write
kernels, then D2H of the bytes) on the cfg2 join's 5.3M matches, against the
reference writer's per-line cost (cli.py:99-108, numpy) on a 200k-line sample."""
import os, sys, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import numpy as np, torch
from paper_2312_01476_b200 import device as D, datagen
from paper_2312_01476_b200.matchio import format_columns_device, format_matches
import fmt_oracle as F
dev = torch.device("cuda:0")
(L, S), c = datagen.config_vectors("cfg2")
m = D.join_prepared(D.prepare(torch.from_numpy(L).to(dev)), D.prepare(torch.from_numpy(S).to(dev)), c["theta"])
print("matches", m.n_matches)
for _ in range(3): out = format_columns_device(m.lefts, m.rights, m.sims)
ts = []
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    out = format_columns_device(m.lefts, m.rights, m.sims)
    e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
nb = out.numel()
print(f"GPU format (layout+scan+write, incl. one sync): median {statistics.median(ts):.3f} ms, {nb/1e6:.1f} MB, {nb/statistics.median(ts)/1e6:.1f} GB/s of text")
ts = []
for _ in range(5):
    t0 = time.perf_counter(); b = format_matches(m); ts.append(time.perf_counter() - t0)
print(f"format_matches (device columns -> host bytes): median {1e3*statistics.median(ts):.2f} ms")
lo, ro, so = m.to_host()
k = 200_000
t0 = time.perf_counter(); ref = F.matches_file_reference(lo[:k], ro[:k], so[:k]); dt = time.perf_counter() - t0
print(f"reference writer: {1e6*dt/k:.2f} us/line -> {dt/k*m.n_matches:.1f} s for the cfg2 file; sample equal: {b[:len(ref)] == ref}")
