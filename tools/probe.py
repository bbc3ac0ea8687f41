"""Quick GPU probe: parity of the fused join vs the CPU oracle, then timing."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2312_01476_b200 import device as D, datagen
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import oracle as O

def check(nl, nr, dim, theta, C=200, sigma=0.5, seed=1):
    L, S = datagen.clustered_pair(nl, nr, dim, C, sigma, seed)
    Lt, St = torch.from_numpy(L).cuda(), torch.from_numpy(S).cuda()
    PL, PS = D.prepare(Lt), D.prepare(St)
    Ln, _ = O.normalize_rows(L); Sn, _ = O.normalize_rows(S)
    ok_norm = np.array_equal(PL.f32.cpu().numpy().view(np.uint32), Ln.view(np.uint32)) and \
              np.array_equal(PS.f32.cpu().numpy().view(np.uint32), Sn.view(np.uint32))
    m = D.join_prepared(PL, PS, theta)
    lo, ro, so = m.to_host()
    rl, rr, rs = O.join_normalized(Ln, Sn, theta, threads=8)
    same = (np.array_equal(lo, rl) and np.array_equal(ro, rr) and np.array_equal(so.view(np.uint32), rs.view(np.uint32)))
    print(f"nl={nl} nr={nr} d={dim} th={theta}: norm_bitexact={ok_norm} gpu={len(lo)} oracle={len(rl)} cand={m.n_candidates} retries={m.retries} grid={m.grid} bitexact={same}", flush=True)
    if not same:
        a = set(zip(lo.tolist(), ro.tolist())); b = set(zip(rl.tolist(), rr.tolist()))
        print("  only_gpu", list(a - b)[:5], "only_oracle", list(b - a)[:5], flush=True)
        if len(lo) == len(rl):
            d = np.nonzero(so != rs)[0]; print("  sim diffs", len(d), d[:5])
    return same

torch.cuda.init()
print(torch.cuda.get_device_name(0), flush=True)
allok = True
for args in [(300, 500, 100, 0.8), (1000, 1000, 100, 0.5), (257, 129, 64, 0.7), (50, 2000, 16, 0.9), (2000, 3000, 100, 0.8), (700, 900, 4, 0.95), (64, 64, 100, -1.0)]:
    allok &= check(*args)
print("ALLOK", allok, flush=True)

# timing at cfg2 shape
(L, S), c = datagen.config_vectors("cfg2")
Lt, St = torch.from_numpy(L).cuda(), torch.from_numpy(S).cuda()
PL, PS = D.prepare(Lt), D.prepare(St)
m = D.join_prepared(PL, PS, 0.8)
print("cfg2 matches", m.n_matches, "cand", m.n_candidates, "retries", m.retries, flush=True)
for it in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    m = D.join_prepared(PL, PS, 0.8)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"cfg2 join {1e3*(t1-t0):.2f} ms -> {1e11/(t1-t0):.3e} pairs/s", flush=True)
torch.cuda.synchronize(); t0 = time.perf_counter()
PL2 = D.prepare(Lt); PS2 = D.prepare(St)
torch.cuda.synchronize(); t1 = time.perf_counter()
print(f"prepare both {1e3*(t1-t0):.2f} ms", flush=True)
