"""Multi-rank orchestration of the R-sharded join on CPU (gloo, world 2).

The per-rank join is the CPU oracle here (test stand-in); what is tested is
the sharding, the broadcast of S, offset shifting and rank-order
concatenation, which must reproduce the single-process canonical result.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_join(R_shard, S, theta, left_base, band):
    import oracle as O
    lo, ro, so = O.join_raw(R_shard.numpy(), S.numpy(), theta)
    return lo + np.uint64(left_base), ro, so


def _worker(rank, world, port, L, S_full, theta, q):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.dirname(here))
    sys.path.insert(0, os.path.join(os.path.dirname(here), "oracle"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2312_01476_b200 import multigpu as MG
    r0, r1 = MG.shard_range(len(L), rank, world)
    S = torch.from_numpy(S_full) if rank == 0 else torch.zeros(S_full.shape, dtype=torch.float32)
    cols = MG.sharded_join(torch.from_numpy(L[r0:r1]), S, theta, r0, join_fn=_oracle_join)
    assert torch.equal(S, torch.from_numpy(S_full))       # broadcast delivered S
    full = MG.gather_to_root(cols)
    if rank == 0:
        q.put(tuple(a.copy() for a in full))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_join_concat_is_canonical(world):
    import oracle as O
    from paper_2312_01476_b200 import datagen
    L, S = datagen.clustered_pair(301, 257, 32, 20, 0.5, seed=3)
    theta = 0.6
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, L, S, theta, q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    want = O.join_raw(L, S, theta)
    assert len(want[0]) > 0
    for a, b in zip(got, want):
        assert np.array_equal(a.view(np.uint32) if a.dtype == np.float32 else a,
                              b.view(np.uint32) if b.dtype == np.float32 else b)


def test_shard_range_covers():
    from paper_2312_01476_b200.multigpu import shard_range
    for n in (0, 1, 7, 100, 100_003):
        for w in (1, 2, 3, 8):
            rs = [shard_range(n, r, w) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))


def _chunk_worker(rank, world, port, S_full, q):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.dirname(here))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2312_01476_b200 import device as D, multigpu as MG
    S = torch.from_numpy(S_full.copy()) if rank == 0 else torch.zeros(S_full.shape,
                                                                     dtype=torch.float32)
    spans = D._stream_chunks(S.shape[0], 5)
    arrive = MG.broadcast_chunks(S, spans)
    ok = True
    for r0, r1 in spans:          # the streamed join's order: chunk by chunk
        arrive(r0, r1)
        ok &= bool(torch.equal(S[r0:r1], torch.from_numpy(S_full[r0:r1])))
    ok &= bool(torch.equal(S, torch.from_numpy(S_full)))
    q.put((rank, ok, [tuple(s) for s in spans]))
    dist.destroy_process_group()


def test_chunked_broadcast_arrives_in_order():
    """The streamed sharded join's S broadcast (multigpu.broadcast_chunks):
    every span is complete on every rank once arrive() returns, spans tile S
    on 512-row boundaries."""
    S = np.random.default_rng(5).standard_normal((2600, 8), dtype=np.float32)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_chunk_worker, args=(r, 2, port, S, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, ok, spans in res:
        assert ok, rank
        assert spans[0][0] == 0 and spans[-1][1] == len(S)
        assert all(a[1] == b[0] and a[1] % 512 == 0 for a, b in zip(spans, spans[1:]))
