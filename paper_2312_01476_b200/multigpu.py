"""R-sharded multi-GPU join (BASELINE.json north star item 5).

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch).  The
paper's own decomposition partitions along tuple lines (PAPER.md:198-201,
330): rank r owns the contiguous left rows [r0, r1) and the
whole right relation, which the root broadcasts once per join.  Each (R-shard
x S) join is independent -- there is no reduction -- and because every rank
emits its shard's matches in canonical (left, right) order with offsets
shifted by r0, concatenating the per-rank MatchSets in rank order is the
canonical MatchSet of the whole join (core.py:196-213 semantics).

The join itself is pluggable (``join_fn``) so the orchestration is testable on
CPU with the gloo backend; the default runs the device pipeline.
"""

from __future__ import annotations

from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np
import torch
import torch.distributed as dist


def shard_range(n: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous balanced row range of `rank` (the reference's outer-row
    bounds formula, join.py:263-264)."""
    return n * rank // world, n * (rank + 1) // world


def world() -> Tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


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


def concat_shards(parts: Sequence[Tuple[np.ndarray, np.ndarray, np.ndarray]]
                  ) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
    """Concatenate per-rank canonical match columns in rank order."""
    parts = [p for p in parts if len(p[0])]
    if not parts:
        return (np.empty(0, np.uint64), np.empty(0, np.uint64), np.empty(0, np.float32))
    return tuple(np.concatenate([p[k] for p in parts]) for k in range(3))


def gather_to_root(cols: Tuple[np.ndarray, np.ndarray, np.ndarray], group=None
                   ) -> Optional[Tuple[np.ndarray, np.ndarray, np.ndarray]]:
    """Collect every rank's host match columns on rank 0 (object gather)."""
    r, w = world()
    if w == 1:
        return cols
    out: List = [None] * w if r == 0 else None
    dist.gather_object(cols, out, dst=0, group=group)
    return concat_shards(out) if r == 0 else None
