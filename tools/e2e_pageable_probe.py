"""cfg2 end to end from PAGEABLE numpy inputs (tensor_join_vectors): wall
time per call (median of 5 after 2 warm-ups) for the pinned bounce ring's
settings in the environment (SJB_BOUNCE_THREADS / SLOT_MB / SLOTS), and the
pinned-input time beside it."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2312_01476_b200 import build, datagen  # noqa: E402
build.build()
from paper_2312_01476_b200.join import tensor_join_vectors  # noqa: E402

(L, S), c = datagen.config_vectors("cfg2")
dev = torch.device("cuda", 0)


def timed(a, b):
    for _ in range(2):
        tensor_join_vectors(a, b, c["theta"], device=dev)
    ts = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ms, _ = tensor_join_vectors(a, b, c["theta"], device=dev)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts) * 1e3, len(ms)


env = {k: os.environ.get(k) for k in ("SJB_BOUNCE_THREADS", "SJB_BOUNCE_SLOT_MB", "SJB_BOUNCE_SLOTS")}
t, n = timed(L, S)
print(f"pageable {env}: {t:.1f} ms ({n} matches)", flush=True)
if os.environ.get("PROBE_PINNED"):
    t, n = timed(torch.from_numpy(L).pin_memory(), torch.from_numpy(S).pin_memory())
    print(f"pinned: {t:.1f} ms", flush=True)
