"""Time prepare + join on several BASELINE configs (device-resident)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2312_01476_b200 import device as D, datagen

def run(name, L, S, theta, iters=3):
    Lt, St = torch.from_numpy(L).cuda(), torch.from_numpy(S).cuda()
    pl, pr = D.prepare(Lt), D.prepare(St)
    m = D.join_prepared(pl, pr, theta)
    ts = []
    for _ in range(iters):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        pl, pr = D.prepare(Lt), D.prepare(St)
        m = D.join_prepared(pl, pr, theta)
        torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    t = min(ts)
    pairs = L.shape[0] * S.shape[0]
    print(f"{name:24s} theta={theta:5.2f} {1e3*t:8.2f} ms  {pairs/t:.3e} pairs/s  matches={m.n_matches} "
          f"cand={m.n_candidates} ({m.n_matches/t:.3e} out/s)", flush=True)

(L, S), c = datagen.config_vectors("cfg1")
run("cfg1 10k x 10k", L, S, 0.8)
(L, S), c = datagen.config_vectors("cfg5")
for th in (0.95, 0.8, 0.6, 0.4):
    run("cfg5 200k x 200k", L, S, th)
