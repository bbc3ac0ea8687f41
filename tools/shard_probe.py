"""Per-rank device work of the strong-scaling bench on one GPU, for N = 1, 2,
4, 8: what rank 0 does in multigpu.sharded_join_owned apart from waiting
for the all-gathers -- prepare its R shard (|R|/N rows), prepare ITS pieces
of S (1/N of S, piece layout of N ranks), filter every round of S on the
reduced grid (SMs - NCCL reserve), finish.  The other ranks' prepared
pieces are put in place before the timed region (on N GPUs they arrive by
NCCL while the filter runs; one GPU cannot run ranks that wait on each
other, so the transfer is not measured here).  The ratio
(step at N=1) / (N * step at N) bounds the strong-scaling efficiency from
the per-rank compute side.  CUDA events, medians of 10 after 3 warm-ups."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2312_01476_b200 import _lib, build, datagen  # noqa: E402
build.build()
from paper_2312_01476_b200 import device as D  # noqa: E402
from paper_2312_01476_b200 import multigpu as MG  # noqa: E402

(L, S), c = datagen.config_vectors("cfg2")
dev = torch.device("cuda", 0)
Ld, Sd = torch.from_numpy(L).to(dev), torch.from_numpy(S).to(dev)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
sms = int(_lib.lib().sjb_sm_count(0))
reserve = MG.nccl_reserve_sms()
base = None
worlds = [int(w) for w in os.environ.get("PROBE_WORLDS", "1,2,4,8").split(",")]
for world in worlds:
    r0, r1 = MG.shard_range(L.shape[0], 0, world)
    R = Ld[r0:r1]
    lay = MG.piece_layout(S.shape[0], world)
    PR = D.empty_prepared(S.shape[0], S.shape[1], dev, rows=lay.rows)
    for k in range(world):                       # every rank's pieces, in place
        for _, a, b in lay.owned(k):
            D.prepare_into(Sd[a:b], PR, a)
    mine = lay.owned(0)
    grid = sms - reserve if world > 1 and reserve > 0 else 0

    def rank0_step():
        PL = D.prepare(R)
        for _, a, b in mine:                     # rank 0 prepares only its pieces
            D.prepare_into(Sd[a:b], PR, a)
        sess = D.JoinSession(PL, PR, c["theta"], None, r0)
        for j in range(lay.rounds):                # as multigpu.sharded_join_owned
            sess.filter_rows(*lay.round_rows(j), launch_grid=0 if j == lay.rounds - 1 else grid)
        return sess.finish().result()

    for _ in range(3):
        rank0_step()
    ts = []
    for _ in range(10):
        torch.cuda.synchronize()
        ev[0].record()
        m = rank0_step()
        ev[1].record()
        torch.cuda.synchronize()
        ts.append(ev[0].elapsed_time(ev[1]))
    t = statistics.median(ts)
    base = base or t
    print(f"N={world}: rank-0 shard {r1 - r0} x {S.shape[0]} (own S pieces "
          f"{lay.local_rows(0)} rows, {lay.rounds} rounds, grid {grid or sms}): {t:.2f} ms "
          f"per step; compute-side efficiency {base / (world * t):.3f}", flush=True)
