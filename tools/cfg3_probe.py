"""cfg3 end to end on one GPU: 200k + 200k strings -> FastText-style subword
embedding on the device (2M x 100 bucket table) -> tensor_join, theta 0.85.
Times the public operator (tensor_join with a SubwordModel) and its parts."""
import os, sys, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2312_01476_b200 import RawRelation, SubwordModel, tensor_join, datagen
from paper_2312_01476_b200 import device as D

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
t0 = time.perf_counter()
left, right = datagen.strings(n, n, 0.3, seed=0)
print(f"strings: {time.perf_counter() - t0:.2f} s", flush=True)
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
table = torch.randn((2_000_000, 100), generator=g, device=dev) * (1.0 / 10.0)
model = SubwordModel(table)
L, R = RawRelation("left", left), RawRelation("right", right)

def embed_only():
    pl = D.subword_rows(left, table, 3, 6, prepared=True)
    pr = D.subword_rows(right, table, 3, 6, prepared=True)
    torch.cuda.synchronize()
    return pl, pr

for _ in range(2):
    embed_only()
ts = []
for _ in range(5):
    a = time.perf_counter(); D.pack_tokens(left, dev); D.pack_tokens(right, dev); ts.append(time.perf_counter() - a)
print(f"host token packing + byte H2D (both relations): median {1e3*statistics.median(ts):.2f} ms", flush=True)
b, o = D.pack_tokens(left, dev)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
import ctypes
from paper_2312_01476_b200 import _lib
f32 = torch.empty((n, 100), device=dev); op = torch.empty(D.operand_elems(n, 100), dtype=torch.bfloat16, device=dev)
rep = torch.zeros(1, dtype=torch.int64, device=dev); re, te = D._err_buffers(n, dev)
ks = []
for _ in range(5):
    e0.record()
    _lib.check(_lib.lib().sjb_subword_embed(D._vp(b), D._vp(o), n, D._vp(table), table.shape[0], 100, 3, 6, 1,
               D._vp(f32), D._vp(op), D._vp(rep), D._vp(re), D._vp(te), D._stream(dev)), "subword")
    e1.record(); torch.cuda.synchronize(); ks.append(e0.elapsed_time(e1))
print(f"subword_embed kernel (one relation, {n} strings): median {statistics.median(ks):.3f} ms", flush=True)
ts = []
for _ in range(5):
    torch.cuda.synchronize(); a = time.perf_counter(); pl, pr = embed_only(); ts.append(time.perf_counter() - a)
print(f"embed+normalise (incl. token packing + H2D of bytes): median {1e3*statistics.median(ts):.2f} ms", flush=True)
for _ in range(2):
    D.join_prepared(pl, pr, 0.85)
ts = []
for _ in range(5):
    torch.cuda.synchronize(); a = time.perf_counter(); m = D.join_prepared(pl, pr, 0.85); torch.cuda.synchronize(); ts.append(time.perf_counter() - a)
print(f"join (device-resident): median {1e3*statistics.median(ts):.2f} ms  matches {m.n_matches} cand {m.n_candidates}  "
      f"{n*n/statistics.median(ts):.3e} pairs/s", flush=True)
for _ in range(2):
    tensor_join(L, R, model, 0.85, budget_bytes=64 << 20)
ts = []
for _ in range(5):
    torch.cuda.synchronize(); a = time.perf_counter(); ms, st = tensor_join(L, R, model, 0.85, budget_bytes=64 << 20); ts.append(time.perf_counter() - a)
print(f"tensor_join (strings in, MatchSet out): median {1e3*statistics.median(ts):.2f} ms  matches {len(ms)}  "
      f"{n*n/statistics.median(ts):.3e} pairs/s", flush=True)
