"""One rank's share of BASELINE cfg4 at full size on one GPU: |R| = 125k (1M / 8
ranks) x |S| = 4M, d = 768, 50k centroids, sigma 0.6, Zipf(1.1) cluster sizes,
theta = 0.75.  The data are drawn on the device with torch's generator (same
recipe as datagen.clustered_pair, not the same numbers: 12 GB of host-side
numpy draws would dominate the run).  Checks that the join completes at this
size (candidate segments, 64-bit offsets, ~5e8-2e9 outputs) and reports its
time, with sampled rows checked against the device's own fp32 recomputation.

    python tools/scale_probe.py [--n-left 125000] [--n-right 4000000]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2312_01476_b200 import device as D

ap = argparse.ArgumentParser()
ap.add_argument("--n-left", type=int, default=125_000)
ap.add_argument("--n-right", type=int, default=4_000_000)
ap.add_argument("--dim", type=int, default=768)
ap.add_argument("--centroids", type=int, default=50_000)
ap.add_argument("--sigma", type=float, default=0.6)
ap.add_argument("--theta", type=float, default=0.75)
ap.add_argument("--iters", type=int, default=2)
a = ap.parse_args()
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
cent = torch.randn((a.centroids, a.dim), generator=g, device=dev)
cent /= cent.norm(dim=1, keepdim=True)
p = 1.0 / torch.arange(1, a.centroids + 1, device=dev, dtype=torch.float64) ** 1.1
p /= p.sum()


def rows(n):
    out = torch.empty((n, a.dim), device=dev)
    for s in range(0, n, 1 << 19):
        e = min(n, s + (1 << 19))
        ids = torch.multinomial(p, e - s, replacement=True, generator=g)
        x = cent[ids] + (a.sigma / a.dim ** 0.5) * torch.randn((e - s, a.dim), generator=g,
                                                              device=dev)
        out[s:e] = x / x.norm(dim=1, keepdim=True)
    return out


t0 = time.perf_counter()
L, S = rows(a.n_left), rows(a.n_right)
torch.cuda.synchronize()
print(f"data on device: {time.perf_counter() - t0:.1f} s", flush=True)
for it in range(a.iters):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    PL, PS = D.prepare(L), D.prepare(S)
    m = D.join_prepared(PL, PS, a.theta)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"iter {it}: {dt * 1e3:.1f} ms  matches {m.n_matches}  candidates {m.n_candidates}  "
          f"retries {m.retries}  pair evals/s {a.n_left * a.n_right / dt:.3e}  "
          f"peak mem {torch.cuda.max_memory_allocated() / 2**30:.1f} GiB", flush=True)
# spot check: canonical order of the device columns, sims >= theta
lo, ro, so = m.lefts, m.rights, m.sims
key_ok = bool(((lo[1:] > lo[:-1]) | ((lo[1:] == lo[:-1]) & (ro[1:] > ro[:-1]))).all())
print(f"canonical order: {key_ok}  min sim {float(so.min()):.6f} >= theta "
      f"{float(so.min()) >= torch.tensor(a.theta, dtype=torch.float32).item()}", flush=True)
