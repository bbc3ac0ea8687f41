"""Run prepare + `iters` joins of a config (for ncu launch lists / captures)."""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2312_01476_b200 import device as D, datagen

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", default="cfg2")
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--theta", type=float, default=None)
ap.add_argument("--n-left", type=int, default=None)
ap.add_argument("--n-right", type=int, default=None)
ap.add_argument("--uniform-band", action="store_true")
a = ap.parse_args()
over = {}
if a.n_left: over["n_left"] = a.n_left
if a.n_right: over["n_right"] = a.n_right
(L, S), c = datagen.config_vectors(a.cfg, **over)
theta = a.theta if a.theta is not None else c["theta"]
Lt, St = torch.from_numpy(L).cuda(), torch.from_numpy(S).cuda()
PL, PS = D.prepare(Lt), D.prepare(St)
ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
fl = []
for i in range(a.iters):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    m = D.join_prepared(PL, PS, theta, filter_events=ev, per_row_band=not a.uniform_band)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    fms = ev[0].elapsed_time(ev[1])
    if i > 0:
        fl.append(fms)
    print(f"{a.cfg} iter {i}: {1e3*(t1-t0):.2f} ms (filter {fms:.2f} ms) matches={m.n_matches} "
          f"cand={m.n_candidates} pairs/s={L.shape[0]*S.shape[0]/(t1-t0):.3e}", flush=True)
if fl:
    import statistics
    print(f"{a.cfg} filter median {statistics.median(fl):.3f} ms  min {min(fl):.3f} ms over {len(fl)}",
          flush=True)
