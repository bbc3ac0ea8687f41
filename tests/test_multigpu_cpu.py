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


def _setup(rank, world, port):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.dirname(here))
    sys.path.insert(0, os.path.join(os.path.dirname(here), "oracle"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)


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


# ---- owner-prepared S (multigpu.sharded_join_owned) -------------------------

class _CpuPrepared:
    """Host stand-in for device.PreparedRelation: canonical fp32 rows (oracle
    normalise), an int16 'operand image' (the top half of each fp32), row
    'errors' (row sums) and per-512-row 'tile' maxima, all padded to
    layout.rows rows like the device buffers."""

    def __init__(self, n, rows, dim):
        self.n, self.dim = n, dim
        self.f32 = torch.full((rows, dim), float("nan"))
        self.op = torch.zeros(rows * dim, dtype=torch.int16)
        self.row_err = torch.zeros(rows)
        self.tile_err = torch.zeros(rows // 256)


def _cpu_prepare(raw):
    import oracle as O
    f32, _ = O.normalize_rows(np.ascontiguousarray(raw, dtype=np.float32))
    op = (f32.view(np.int32) >> 16).astype(np.int16).reshape(-1)
    err = f32.sum(axis=1, dtype=np.float32)
    tiles = [err[t:t + 256].max(initial=-np.inf) for t in range(0, len(err), 256)]
    return f32, op, err, np.array(tiles, dtype=np.float32)


class _CpuOps:
    grid = 0          # launch grid of the non-final rounds (device: SMs - NCCL reserve)

    def prepare_left(self, R):
        import oracle as O
        return O.normalize_rows(R.numpy())[0]

    def alloc_right(self, layout, dim, dev):
        return _CpuPrepared(layout.n, layout.rows, dim)

    def gather_buffers(self, prep, layout):
        return [(prep.f32.view(-1).view(torch.uint8), prep.dim * 4, 1),
                (prep.op.view(torch.uint8), prep.dim * 2, 1),
                (prep.row_err.view(torch.uint8), 4, 1),
                (prep.tile_err.view(torch.uint8), 4, 256)]

    def prepare_piece(self, raw, prep, r0):
        m = raw.shape[0]
        if m == 0:
            return
        f32, op, err, tiles = _cpu_prepare(raw.numpy())
        prep.f32[r0:r0 + m] = torch.from_numpy(f32)
        prep.op[r0 * prep.dim:(r0 + m) * prep.dim] = torch.from_numpy(op)
        prep.row_err[r0:r0 + m] = torch.from_numpy(err)
        prep.tile_err[r0 // 256:r0 // 256 + len(tiles)] = torch.from_numpy(tiles)

    def session(self, PL, PR, theta, band, left_base):
        return _CpuSession(PL, PR, theta, left_base)


class _CpuSession:
    def __init__(self, PL, PR, theta, left_base):
        self.PL, self.PR, self.theta, self.base = PL, PR, theta, left_base
        self.parts, self.seen = [], []

    def filter_rows(self, r0, r1, launch_grid=0):
        import oracle as O
        if r1 <= r0:
            return
        self.seen.append((r0, r1))
        S = self.PR.f32[r0:r1].numpy()
        assert not np.isnan(S).any(), "filtered rows that had not arrived"
        lo, ro, so = O.join_normalized(self.PL, S, self.theta)
        self.parts.append((lo, ro + np.uint64(r0), so))

    def finish(self):
        sess = self

        class _Done:
            def result(self):
                lo = np.concatenate([p[0] for p in sess.parts] or [np.empty(0, np.uint64)])
                ro = np.concatenate([p[1] for p in sess.parts] or [np.empty(0, np.uint64)])
                so = np.concatenate([p[2] for p in sess.parts] or [np.empty(0, np.float32)])
                order = np.lexsort((ro, lo))
                return lo[order] + np.uint64(sess.base), ro[order], so[order]
        return _Done()


def _owned_worker(rank, world, port, L, S_full, theta, rounds, q):
    _setup(rank, world, port)
    from paper_2312_01476_b200 import multigpu as MG
    lay = MG.piece_layout(len(S_full), world, rounds, align=512)
    r0, r1 = MG.shard_range(len(L), rank, world)
    S_local = torch.from_numpy(MG.local_pieces(S_full, lay, rank))
    cols, PR = MG.sharded_join_owned(torch.from_numpy(L[r0:r1]), S_local, lay, theta, r0,
                                     ops=_CpuOps())
    f32, op, err, tiles = _cpu_prepare(S_full)
    n = len(S_full)
    ok = bool(np.array_equal(PR.f32[:n].numpy().view(np.uint32), f32.view(np.uint32)))
    ok &= bool(np.array_equal(PR.op[:n * S_full.shape[1]].numpy(), op))
    ok &= bool(np.array_equal(PR.row_err[:n].numpy(), err))
    ok &= bool(np.array_equal(PR.tile_err[:len(tiles)].numpy(), tiles))
    full = MG.gather_to_root(cols)
    q.put((rank, ok, S_local.shape[0], None if full is None else tuple(a.copy() for a in full)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,rounds,n_right", [(2, 2, 2600), (4, 0, 5000), (4, 3, 700)])
def test_owner_prepared_sharded_join(world, rounds, n_right):
    """Each rank prepares only its own pieces of S; the per-round in-place
    all-gathers assemble the full prepared S (bitwise) on every rank, no rank
    filters rows before they arrived, and the rank-local results concatenate
    to the single-process canonical join (multigpu.sharded_join_owned)."""
    import oracle as O
    from paper_2312_01476_b200 import datagen
    from paper_2312_01476_b200 import multigpu as MG
    L, S = datagen.clustered_pair(203, n_right, 16, 12, 0.5, seed=world + n_right)
    theta = 0.7
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_owned_worker, args=(r, world, port, L, S, theta, rounds, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=180) for _ in range(world)), key=lambda x: x[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    lay = MG.piece_layout(n_right, world, rounds)
    assert sum(r[2] for r in res) == n_right           # every S row held by exactly one rank
    assert [r[2] for r in res] == [lay.local_rows(k) for k in range(world)]
    assert all(r[1] for r in res), "gathered prepared S differs from a single-process prepare"
    want = O.join_raw(L, S, theta)
    got = res[0][3]
    assert len(want[0]) > 0
    assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])
    assert np.array_equal(got[2].view(np.uint32), want[2].view(np.uint32))


def test_piece_layout_covers():
    from paper_2312_01476_b200.multigpu import piece_layout
    for n in (0, 1, 511, 512, 5000, 1_000_000):
        for w in (1, 2, 3, 8):
            lay = piece_layout(n, w)
            assert all(p % 512 == 0 for p in lay.pieces) and lay.rows >= n
            assert list(lay.pieces) == sorted(lay.pieces)
            spans = [lay.piece_rows(j, k) for j in range(lay.rounds) for k in range(w)]
            real = [(a, b) for a, b in spans if b > a]
            assert sum(b - a for a, b in real) == n
            assert all(a[1] == b[0] for a, b in zip(real, real[1:]))
            assert sum(lay.local_rows(k) for k in range(w)) == n
