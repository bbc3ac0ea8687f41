"""Small joins through every device path, for compute-sanitizer runs:
d <= 128 fused / deferred recheck, CTA-pair filter, wide (d = 768) filter +
staged recheck, streamed join, cosine_vm.  Exits non-zero on a mismatch."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import numpy as np, torch
import oracle as O
from paper_2312_01476_b200 import datagen, device as D
from paper_2312_01476_b200.linalg import cosine_vm

dev = torch.device("cuda:0")
only = sys.argv[1] if len(sys.argv) > 1 else "all"


def check(L, S, theta, **kw):
    m = D.join_prepared(D.prepare(torch.from_numpy(L).to(dev)),
                        D.prepare(torch.from_numpy(S).to(dev)), theta, **kw)
    lo, ro, so = m.to_host()
    wl, wr, ws = O.join_raw(L, S, theta, threads=8)
    assert np.array_equal(lo, wl) and np.array_equal(ro, wr), (L.shape, S.shape, theta)
    assert np.array_equal(so.view(np.uint32), ws.view(np.uint32))


L, S = datagen.clustered_pair(700, 1300, 100, 40, 0.5, 1)
if only in ("all", "fused"):
    os.environ["SJB_RECHECK"] = "fused"; check(L, S, 0.7); check(L, S, 0.7, cand_cap=600)
if only in ("all", "deferred"):
    os.environ["SJB_RECHECK"] = "deferred"; check(L, S, 0.5)
os.environ.pop("SJB_RECHECK", None)
if only in ("all", "pair"):
    os.environ["SJB_FILTER"] = "pair"; check(L, S, 0.7); os.environ.pop("SJB_FILTER")
if only in ("all", "wide"):
    Lw, Sw = datagen.clustered_pair(300, 700, 768, 20, 0.6, 2, zipf=1.1)
    check(Lw, Sw, 0.75)
if only in ("all", "streamed"):
    m, _ = D.join_streamed(D.prepare(torch.from_numpy(L).to(dev)), torch.from_numpy(S), 0.7,
                           chunks=3)
    lo, ro, so = m.to_host()
    wl, wr, ws = O.join_raw(L, S, 0.7, threads=8)
    assert np.array_equal(lo, wl) and np.array_equal(so.view(np.uint32), ws.view(np.uint32))
if only in ("all", "cosine"):
    a = np.random.default_rng(3).standard_normal(100).astype(np.float32)
    got = cosine_vm(a, S)
    want = np.divide(O.dots_vm(a, S), np.multiply(O.row_norms(a.reshape(1, -1))[0],
                                                  O.row_norms(S), dtype=np.float32),
                     dtype=np.float32)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
torch.cuda.synchronize()
print("sanitize paths ok:", only)
