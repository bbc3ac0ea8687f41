"""R-sharded multi-GPU join (BASELINE.json north star item 5).

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch).  The
paper's own decomposition partitions along tuple lines (PAPER.md:198-201,
330): rank r owns the contiguous left rows [r0, r1) -- the
reference's outer-row bounds formula (join.py:263-264) -- and joins them
against the whole right relation S.  Each (R-shard x S) join is independent,
so there is no reduction: every rank emits its shard's matches in canonical
(left, right) order with offsets shifted by r0, and the per-rank results,
concatenated in rank order, are the canonical MatchSet of the whole join
(core.py:196-213 semantics).  Results stay rank-local (device columns, or
the rank's pinned host copy); nothing funnels them through one process.

S reaches every rank PREPARED, and each row is prepared exactly once in the
whole job (``sharded_join_owned``):

* S is cut into rounds of ``world`` equal pieces (multiples of 512 rows, so
  a piece is whole operand tiles; the rounds grow geometrically so the
  filter waits only for the small first one); piece k of round j belongs to
  rank k.  Rank k holds the raw rows of its own pieces.
* Each rank normalises its pieces (canonical fp32 rows, operand image, row
  and tile rounding errors) straight into its slot of the full prepared
  buffers, then round j is ONE in-place all-gather per buffer: the round's
  pieces are contiguous in S, so the world's pieces land in row order.
* Every rank filters round j's rows as soon as its all-gather has landed
  (device.JoinSession), while rounds j+1.. are still on the wire.  While
  later gathers are in flight the filter launches on SMs - reserve CTAs so
  NCCL's kernels always have SMs beside the persistent filter; the last
  round runs on the whole GPU.

``sharded_join_streamed`` (rank 0 holds raw S and broadcasts it in row
chunks; every rank normalises all of S) is kept for callers whose S exists on
one rank only.

The per-rank compute is pluggable (``ops``) so the orchestration -- piece
ownership, the all-gathers, the round order and the result assembly -- is
tested on CPU with the gloo backend (tests/test_multigpu_cpu.py).
"""

from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np
import torch
import torch.distributed as dist

ALIGN = 512          # rows: an operand tile pair (device.PreparedRelation.rows)


def shard_range(n: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous balanced row range of `rank` (the reference's outer-row
    bounds formula, join.py:263-264)."""
    return n * rank // world, n * (rank + 1) // world


def world() -> Tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


@dataclass(frozen=True)
class PieceLayout:
    """S cut into rounds of `world` equal pieces: round j's pieces have
    pieces[j] rows each (a multiple of 512) and are contiguous in S, piece k
    of round j belonging to rank k.  Rows beyond n are padding (never
    prepared, never joined)."""

    n: int
    world: int
    pieces: Tuple[int, ...]

    @property
    def rounds(self) -> int:
        return len(self.pieces)

    @property
    def rows(self) -> int:
        """Padded row count of the prepared buffers (every piece full size)."""
        return self.world * sum(self.pieces)

    def round_start(self, j: int) -> int:
        return self.world * sum(self.pieces[:j])

    def piece_rows(self, j: int, k: int) -> Tuple[int, int]:
        r0 = self.round_start(j) + k * self.pieces[j]
        return r0, max(r0, min(self.n, r0 + self.pieces[j]))

    def round_rows(self, j: int) -> Tuple[int, int]:
        r0 = self.round_start(j)
        return r0, max(r0, min(self.n, r0 + self.world * self.pieces[j]))

    def owned(self, rank: int) -> List[Tuple[int, int, int]]:
        """(round, r0, r1) of every piece `rank` owns (r1 - r0 may be 0)."""
        return [(j, *self.piece_rows(j, rank)) for j in range(self.rounds)]

    def local_rows(self, rank: int) -> int:
        """Real rows `rank` holds (the sum of its pieces)."""
        return sum(r1 - r0 for _, r0, r1 in self.owned(rank))


def piece_layout(n: int, world: int, rounds: int = 0, growth: float = 1.5,
                 align: int = ALIGN) -> PieceLayout:
    """Pieces for the owner-prepared all-gather, growing geometrically by
    `growth` per round: the filter waits only for round 0's gather, and each
    later round's gather (time ~ rows) runs behind the previous round's
    filter (time ~ rows / world ... rows), which is longer once
    growth <= filter time per row / gather time per row.  rounds=0 picks up
    to 4 rounds, fewer when S is small (no round below one 512-row piece per
    rank).  Four rounds: each filter launch of a round costs ~0.05 ms of
    launch and tail at cfg2 / 8 ranks (tools/shard_probe.py: 2.2 ms per rank
    step with 1 or 4 rounds, 2.6-2.8 ms with 8)."""
    world = max(1, int(world))
    unit = world * align
    if rounds <= 0:
        rounds = int(os.environ.get("SJB_SHARD_ROUNDS", "0")) or max(1, min(4, n // (4 * unit)))
    growth = float(os.environ.get("SJB_SHARD_GROWTH", growth))
    weights = [growth ** j for j in range(rounds)]
    total = sum(weights)
    pieces = []
    covered = 0
    for j, wgt in enumerate(weights):
        want = n - covered if j == rounds - 1 else int(n * wgt / total)
        per_rank = -(-max(want, 1) // world)
        pieces.append(-(-per_rank // align) * align)
        covered += pieces[-1] * world
        if covered >= n:
            break
    return PieceLayout(n, world, tuple(pieces))


def local_pieces(S: np.ndarray, layout: PieceLayout, rank: int) -> np.ndarray:
    """The raw rows of `rank`'s pieces, concatenated in round order (what
    that rank holds when the job starts)."""
    parts = [S[r0:r1] for _, r0, r1 in layout.owned(rank)]
    if not parts:
        return S[:0]
    return np.ascontiguousarray(np.concatenate(parts)) if len(parts) > 1 else parts[0]


def _gather_round(bufs: Sequence[Tuple[torch.Tensor, int, int]], layout: PieceLayout, j: int,
                  rank: int, group=None) -> list:
    """Queue round j's in-place all-gathers.  bufs: (flat byte tensor, bytes,
    per rows) -- `bytes` per `rows` S rows; a buffer's round-j slice is
    contiguous and its rank-k slice is the piece of rank k."""
    works = []
    for flat, nbytes, rows in bufs:
        per_piece = nbytes * layout.pieces[j] // rows
        base = nbytes * layout.round_start(j) // rows
        out = flat[base:base + layout.world * per_piece]
        inp = out[rank * per_piece:(rank + 1) * per_piece]
        works.append(dist.all_gather_into_tensor(out, inp, group=group, async_op=True))
    return works


class DeviceOps:
    """The device side of sharded_join_owned (libsjb200.so kernels)."""

    def __init__(self, grid: int = 0):
        self.grid = grid

    def prepare_left(self, R_shard: torch.Tensor):
        from . import device as D
        return D.prepare(R_shard)

    def alloc_right(self, layout: PieceLayout, dim: int, dev):
        from . import device as D
        return D.empty_prepared(layout.n, dim, dev, rows=layout.rows)

    def gather_buffers(self, prep, layout: PieceLayout):
        """(flat byte view, bytes, per rows) of every prepared buffer (tile
        errors: 4 bytes per 256-row tile; pieces are whole tile pairs)."""
        from . import device as D
        dim = prep.dim
        return [(prep.f32.view(-1).view(torch.uint8), dim * 4, 1),
                (prep.op.view(torch.uint8), D.kpad(dim) * 2, 1),
                (prep.row_err.view(torch.uint8), 4, 1),
                (prep.tile_err.view(torch.uint8), 4, D.TILE_ROWS)]

    def prepare_piece(self, raw: torch.Tensor, prep, r0: int) -> None:
        from . import device as D
        D.prepare_into(raw, prep, r0)

    def session(self, PL, PR, theta: float, band, left_base: int):
        from . import device as D
        return D.JoinSession(PL, PR, theta, band, left_base)


def nccl_reserve_sms() -> int:
    """SMs the streamed filter leaves free for NCCL's collective kernels:
    NCCL_MAX_CTAS when set (bench.py sets it), else 16."""
    return int(os.environ.get("NCCL_MAX_CTAS", "16"))


def sharded_join_owned(R_shard, S_local, layout: PieceLayout, theta: float, left_base: int,
                       group=None, band: Optional[float] = None, ops=None, sync: bool = True):
    """This rank's share of the R-sharded join with owner-prepared S.

    R_shard: this rank's left rows (device); S_local: the raw rows of this
    rank's pieces of S in round order (layout.local_rows(rank) rows).  Each
    rank prepares only its own pieces; round j's prepared rows are one
    in-place all-gather per buffer, and every rank filters a round as soon as
    it has landed.  Returns (matches, prepared S): the rank-local matches
    (device.DeviceMatches with left offsets shifted by left_base; a
    PendingJoin when sync=False) and the full prepared S, resident on this
    rank for further joins."""
    rank, w = world()
    if w != layout.world:
        raise ValueError(f"layout is for {layout.world} ranks, the world has {w}")
    if ops is None:
        from . import _lib
        sms = int(_lib.lib().sjb_sm_count(R_shard.device.index or 0))
        ops = DeviceOps(grid=max(1, sms - nccl_reserve_sms()) if w > 1 else 0)
    dim = R_shard.shape[1]
    if S_local.shape[0] != layout.local_rows(rank) or S_local.shape[1] != dim:
        raise ValueError(f"rank {rank} holds {tuple(S_local.shape)}, layout expects "
                         f"({layout.local_rows(rank)}, {dim})")
    PL = ops.prepare_left(R_shard)
    PR = ops.alloc_right(layout, dim, R_shard.device)
    off = 0
    for _, r0, r1 in layout.owned(rank):                 # prepare my pieces, once
        ops.prepare_piece(S_local[off:off + (r1 - r0)], PR, r0)
        off += r1 - r0
    bufs = ops.gather_buffers(PR, layout)
    works = []
    if w > 1:
        for j in range(layout.rounds):                   # all queued now, in order
            works.append(_gather_round(bufs, layout, j, rank, group))
    session = ops.session(PL, PR, theta, band, left_base)
    for j in range(layout.rounds):
        for wk in (works[j] if works else ()):
            wk.wait()                                    # the stream waits, not the host
        # while later rounds' gathers are in flight the filter leaves NCCL its
        # SMs; the last round has nothing in flight and takes the whole GPU
        last = j == layout.rounds - 1
        session.filter_rows(*layout.round_rows(j), launch_grid=0 if last else ops.grid)
    pending = session.finish()
    return (pending.result() if sync else pending), PR


def gather_right_raw(S_local: torch.Tensor, layout: PieceLayout, group=None) -> torch.Tensor:
    """The whole right relation on every rank from each rank's raw pieces
    (layout order): one in-place all-gather per round.  For relations whose
    preparation is cheap next to the join (cfg4: bf16 rows, d = 768 -- the
    raw bf16 rows are half the bytes of the prepared fp32 rows, and each rank
    prepares all of S in ~1% of its join), the raw rows travel and every
    rank prepares locally."""
    rank, w = world()
    dim = S_local.shape[1]
    out = torch.empty((layout.rows, dim), dtype=S_local.dtype, device=S_local.device)
    off = 0
    for _, r0, r1 in layout.owned(rank):
        out[r0:r1].copy_(S_local[off:off + (r1 - r0)])
        off += r1 - r0
    if w > 1:
        flat = out.view(-1).view(torch.uint8)
        per_row = dim * out.element_size()
        for j in range(layout.rounds):
            for wk in _gather_round([(flat, per_row, 1)], layout, j, rank, group):
                wk.wait()
    return out[:layout.n]


# ---- root-broadcast variant (S on one rank) --------------------------------

def broadcast_right(S: torch.Tensor, root: int = 0, group=None, chunk_rows: int = 0) -> torch.Tensor:
    """Broadcast the right relation from `root` in place (all ranks pass a
    tensor of the full shape).  chunk_rows > 0 splits it into row chunks."""
    r, w = world()
    if w == 1:
        return S
    if chunk_rows <= 0 or chunk_rows >= S.shape[0]:
        dist.broadcast(S, src=root, group=group)
        return S
    for s in range(0, S.shape[0], chunk_rows):
        dist.broadcast(S[s:s + chunk_rows], src=root, group=group)
    return S


def broadcast_chunks(S: torch.Tensor, spans: Sequence[Tuple[int, int]], root: int = 0,
                     group=None) -> Callable[[int, int], None]:
    """Queue one asynchronous broadcast per row span of S (in order, on the
    backend's stream) and return arrive(r0, r1), which makes the caller wait
    for the span starting at r0 (for NCCL: the current CUDA stream waits; the
    host does not block)."""
    r, w = world()
    works = {}
    if w > 1:
        for r0, r1 in spans:
            works[r0] = dist.broadcast(S[r0:r1], src=root, group=group, async_op=True)

    def arrive(r0: int, r1: int) -> None:
        wk = works.pop(r0, None)
        if wk is not None:
            wk.wait()

    return arrive


def _device_join(R_shard: torch.Tensor, S: torch.Tensor, theta: float, left_base: int,
                 band: Optional[float]):
    from . import device as D
    pl = D.prepare(R_shard)
    pr = D.prepare(S)
    return D.join_prepared(pl, pr, theta, band, left_base=left_base)


def sharded_join(R_shard: torch.Tensor, S: torch.Tensor, theta: float, left_base: int,
                 group=None, band: Optional[float] = None,
                 join_fn: Optional[Callable] = None):
    """Broadcast S from rank 0, then join this rank's R shard against it.

    Returns whatever ``join_fn`` returns (default: device.DeviceMatches with
    left offsets already shifted by ``left_base``)."""
    broadcast_right(S, 0, group)
    fn = join_fn or _device_join
    return fn(R_shard, S, theta, left_base, band)


def sharded_join_streamed(R_shard: torch.Tensor, S: torch.Tensor, theta: float, left_base: int,
                          group=None, band: Optional[float] = None, chunks: int = 8):
    """sharded_join with the S broadcast overlapped with the join: S goes out
    from rank 0 in row chunks (NCCL broadcasts queued at once on NCCL's
    stream); each rank normalises and filters chunk k (device.join_chunked)
    as soon as its broadcast has landed, while chunks k+1.. are still in
    flight.  S must be a device tensor of the full shape on every rank (rank
    0's is the source and is left unchanged).  Returns device.DeviceMatches
    with left offsets shifted by ``left_base``."""
    from . import device as D
    pl = D.prepare(R_shard)
    arrive = broadcast_chunks(S, D._stream_chunks(S.shape[0], chunks), root=0, group=group)
    m, _ = D.join_chunked(pl, S, arrive, theta, band, left_base, chunks, inplace=False)
    return m


# ---- result assembly --------------------------------------------------------

def concat_shards(parts: Sequence[Tuple[np.ndarray, np.ndarray, np.ndarray]]
                  ) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
    """Concatenate per-rank canonical match columns in rank order."""
    parts = [p for p in parts if len(p[0])]
    if not parts:
        return (np.empty(0, np.uint64), np.empty(0, np.uint64), np.empty(0, np.float32))
    return tuple(np.concatenate([p[k] for p in parts]) for k in range(3))


def gather_to_root(cols: Tuple[np.ndarray, np.ndarray, np.ndarray], group=None
                   ) -> Optional[Tuple[np.ndarray, np.ndarray, np.ndarray]]:
    """Collect every rank's host match columns on rank 0 in rank order, as
    tensors (counts all-gathered, columns padded to the largest count and
    gathered).  For checks and small results: a production caller keeps the
    rank-local columns (the concatenation in rank order is implicit)."""
    r, w = world()
    if w == 1:
        return cols
    lo, ro, so = cols
    k = torch.tensor([len(lo)], dtype=torch.int64)
    ks = [torch.zeros(1, dtype=torch.int64) for _ in range(w)]
    dist.all_gather(ks, k, group=group)
    kmax = max(int(x) for x in ks)
    packed = torch.zeros((kmax, 3), dtype=torch.int64)
    if len(lo):
        packed[:len(lo), 0] = torch.from_numpy(lo.view(np.int64))
        packed[:len(lo), 1] = torch.from_numpy(ro.view(np.int64))
        packed[:len(lo), 2] = torch.from_numpy(so.view(np.int32).astype(np.int64))
    out = [torch.zeros((kmax, 3), dtype=torch.int64) for _ in range(w)] if r == 0 else None
    dist.gather(packed, out, dst=0, group=group)
    if r != 0:
        return None
    parts = []
    for t, kk in zip(out, ks):
        a = t[:int(kk)].numpy()
        parts.append((a[:, 0].copy().view(np.uint64), a[:, 1].copy().view(np.uint64),
                      a[:, 2].astype(np.int32).view(np.float32)))
    return concat_shards(parts)
