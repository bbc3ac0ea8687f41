"""cfg4-distribution joins (d = 768 bf16, 50k centroids, sigma 0.6,
Zipf(1.1), theta 0.75) on one GPU: time per join (CUDA events, median of
`reps` after one warm-up) for the raw-operand path with canonical and with
tensor similarities, and for the fp32 path; prints matches, candidates and
pairs/s.  Usage: python tools/cfg4_probe.py [n_left] [n_right] [reps] [modes]
(modes: comma list of exact,tensor,fp32)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2312_01476_b200 import build, datagen  # noqa: E402
build.build()
from paper_2312_01476_b200 import device as D  # noqa: E402

nl = int(sys.argv[1]) if len(sys.argv) > 1 else 16_000
nr = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
modes = (sys.argv[4] if len(sys.argv) > 4 else "exact,tensor,fp32").split(",")
(L, S), c = datagen.config_vectors("cfg4", n_left=nl, n_right=nr)
theta = c["theta"]
dev = torch.device("cuda", 0)
bf = lambda x: torch.from_numpy(datagen.bf16_bits(x).view(np.int16)).view(  # noqa: E731
    torch.bfloat16).to(dev)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for mode in modes:
    if mode == "fp32":
        pl, pr = D.prepare(torch.from_numpy(L).to(dev)), D.prepare(torch.from_numpy(S).to(dev))
        sims = "exact"
    else:
        pl, pr = D.prepare_bf16(bf(L)), D.prepare_bf16(bf(S))
        sims = mode
    m = D.join_prepared(pl, pr, theta, sims=sims)
    ts = []
    for _ in range(reps):
        m = None
        torch.cuda.synchronize()
        e0.record()
        m = D.join_prepared(pl, pr, theta, sims=sims)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = statistics.median(ts)
    print(f"{mode}: {nl} x {nr}: {t:.1f} ms, matches {m.n_matches}, candidates "
          f"{m.n_candidates}, {nl * nr / t * 1e3:.3e} pairs/s", flush=True)
    del pl, pr, m
    torch.cuda.empty_cache()
