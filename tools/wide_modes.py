"""Attribute the wide (d > 128) filter's time on a cfg4 slice: the raw-bf16
tensor-sims join timed in the diagnostic modes of the wide filters
(SJB_DEBUG_MODE: 0 full, 1 drain without emission, 2 no drain = MMA + operand
delivery, 20 no operand traffic after the ring filled = MMA + epilogue), for
each filter variant named in VARIANTS (default: the 1-CTA kernel; `mma2`,
`pair` need the A/B build).  Results of modes != 0 are invalid by design;
only the times matter.  CUDA events, median of `reps`.
Usage: python tools/wide_modes.py [n_left] [n_right] [reps]"""
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
variants = os.environ.get("VARIANTS", "single").split(",")
modes = [int(m) for m in os.environ.get("MODES", "0,1,2,20").split(",")]
(L, S), c = datagen.config_vectors("cfg4", n_left=nl, n_right=nr)
theta = c["theta"]
dev = torch.device("cuda", 0)
bf = lambda x: torch.from_numpy(datagen.bf16_bits(x).view(np.int16)).view(  # noqa: E731
    torch.bfloat16).to(dev)
pl, pr = D.prepare_bf16(bf(L)), D.prepare_bf16(bf(S))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
flop = 2.0 * nl * nr * L.shape[1]
for var in variants:
    for k in ("SJB_WIDE_MMA2", "SJB_WIDE_PAIR"):
        os.environ.pop(k, None)
    if var == "mma2":
        os.environ["SJB_WIDE_MMA2"] = "1"
    elif var == "mma2s":   # 256 x 256 pair tiles, two accumulator stages
        os.environ["SJB_WIDE_MMA2"] = "2"
    elif var == "pair":
        os.environ["SJB_WIDE_PAIR"] = "1"
    for mode in modes:
        os.environ["SJB_DEBUG_MODE"] = str(mode)
        try:
            m = D.join_prepared(pl, pr, theta, sims="tensor")
        except Exception as e:  # noqa: BLE001
            print(f"{var} mode {mode}: {e}", flush=True)
            break
        ts = []
        for _ in range(reps):
            m = None
            torch.cuda.synchronize()
            e0.record()
            m = D.join_prepared(pl, pr, theta, sims="tensor")
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        t = statistics.median(ts)
        print(f"{var} mode {mode:2d}: {nl} x {nr}: {t:.2f} ms ({flop / t / 1e9:.0f} TFLOP/s), "
              f"candidates {m.n_candidates}", flush=True)
os.environ.pop("SJB_DEBUG_MODE", None)
