"""Timing of the HBM-bound prep kernels (CUDA events, medians of 20, L2
flushed before each): the subword gather (cfg3: 200k strings against a
2M x 100 table) and its normalise pass, and normalise-and-cast of cfg2's S
(1M x 100).  Prints algorithmic bytes per launch and GB/s."""
import ctypes
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2312_01476_b200 import _lib, build, datagen  # noqa: E402
build.build()
from paper_2312_01476_b200 import device as D  # noqa: E402

dev = torch.device("cuda:0")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


out = {}
left, _ = datagen.strings(200_000, 10, 0.3, seed=0)
n, dim = len(left), 100
g = torch.Generator(device=dev).manual_seed(0)
table = torch.randn((2_000_000, dim), generator=g, device=dev) * 0.1
b, o = D.pack_tokens(left, dev)
lens = (o[1:] - o[:-1]).cpu()
items = int(sum(1 + sum(max(0, int(x) + 2 - gg + 1) for gg in range(3, 7)) for x in lens.tolist()))
f32 = torch.empty((n, dim), device=dev)
op = D.op_empty(n, dim, dev)
rep = torch.zeros(1, dtype=torch.int64, device=dev)
re, te = D._err_buffers(n, dev)
L = _lib.lib()


def subword(prepared):
    _lib.check(L.sjb_subword_embed(D._vp(b), D._vp(o), n, D._vp(table), table.shape[0], dim, 3, 6,
                                   1 if prepared else 0, D._vp(f32), D._vp(op), D._vp(rep),
                                   D._vp(re), D._vp(te), D._stream(dev)), "subword")


gather_bytes = items * dim * 4 + n * dim * 4          # item rows read + mean rows written
t_g = timed(lambda: subword(False))
t_p = timed(lambda: subword(True))
out["subword_gather"] = {"ms": t_g, "strings": n, "items": items,
                         "algorithmic_bytes": gather_bytes, "GBps": gather_bytes / t_g / 1e6}
norm_bytes = n * (4 * dim + 4 * dim + 2 * D.kpad(dim) + 4)
out["subword_prepared"] = {"ms": t_p, "normalise_ms": t_p - t_g,
                           "algorithmic_bytes": gather_bytes + norm_bytes,
                           "GBps": (gather_bytes + norm_bytes) / t_p / 1e6}
(Lv, S), c = datagen.config_vectors("cfg2")
Sd = torch.from_numpy(S).to(dev)
t_n = timed(lambda: D.prepare(Sd))
nb = S.shape[0] * (4 * dim + 4 * dim + 2 * D.kpad(dim) + 4)
out["normalize_cast_cfg2_S"] = {"ms": t_n, "rows": S.shape[0], "algorithmic_bytes": nb,
                                "GBps": nb / t_n / 1e6}
print(json.dumps(out, indent=1))
