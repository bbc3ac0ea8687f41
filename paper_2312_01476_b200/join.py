"""Join operators with the reference's signatures (join.py:88-373), executed
on the B200 path.

``tensor_join`` and ``nlj_prefetch`` keep the reference's arguments, errors,
return types (canonical MatchSet, JoinStats) and model-call accounting.  Both
run the same device pipeline -- prefetch (|R| + |S| model calls), normalise
and cast, fused tensor-core filter, canonical fp32 recheck, canonical order
-- because their outputs are contractually identical (SPEC.md "exactness").
``threads`` and ``budget_bytes`` are validated and recorded exactly as the
reference does; they do not change the device execution (there is no
materialised similarity buffer, so ``peak_buffer_bytes`` reports 0).
"""

from __future__ import annotations

import math
import os
import time
from dataclasses import dataclass
from typing import Optional, Tuple, Union

import numpy as np
import torch

from . import device as D
from .core import EmbeddedRelation, MatchSet, RawRelation, Threshold, check_dims
from .embedding import EmbeddingModel, prepare_relation
from .errors import BudgetTooSmall

# reference constants (join.py:44, 48; cli.py:31)
PREFILTER_BAND = 1e-4
EXEC_CHUNK_ELEMS = 1 << 19
DEFAULT_BUDGET = 64 * 1024 * 1024


@dataclass(frozen=True)
class Tile:
    """Rectangular left-rows x right-rows sub-range (linalg.py:21-38)."""

    left_row_start: int
    left_row_count: int
    right_row_start: int
    right_row_count: int

    def __post_init__(self):
        if self.left_row_count < 1 or self.right_row_count < 1:
            raise ValueError("tile row counts must be >= 1")
        if self.left_row_start < 0 or self.right_row_start < 0:
            raise ValueError("tile offsets must be >= 0")

    @property
    def area(self) -> int:
        return self.left_row_count * self.right_row_count


@dataclass(frozen=True)
class BatchPlan:
    left_block_rows: int
    right_block_rows: int
    tiles: Tuple[Tile, ...]
    buffer_elems: int
    budget_bytes: int


@dataclass(frozen=True)
class JoinStats:
    wall_nanos: int
    model_calls_left: int
    model_calls_right: int
    pairs_compared: int
    matches: int
    peak_buffer_bytes: int
    threads: int
    algo: str
    inner_relation: str

    def to_dict(self) -> dict:
        return {k: getattr(self, k) for k in (
            "wall_nanos", "model_calls_left", "model_calls_right", "pairs_compared", "matches",
            "peak_buffer_bytes", "threads", "algo", "inner_relation")}


def _check_budget(budget_bytes: int) -> None:
    if budget_bytes < 4:
        raise BudgetTooSmall(f"budget {budget_bytes} bytes cannot hold one fp32 cell")


def plan_batches(left_rows: int, right_rows: int, dim: int, budget_bytes: int) -> BatchPlan:
    """Exact-cover grid of near-square blocks under the budget (join.py:88-108)."""
    _check_budget(budget_bytes)
    budget_elems = budget_bytes // 4
    b = math.isqrt(budget_elems)
    lb = max(1, min(b, left_rows))
    rb = max(1, min(budget_elems // lb, right_rows))
    tiles = tuple(Tile(ls, min(lb, left_rows - ls), rs, min(rb, right_rows - rs))
                  for ls in range(0, left_rows, lb) for rs in range(0, right_rows, rb))
    return BatchPlan(lb, rb, tiles, max((t.area for t in tiles), default=0), budget_bytes)


def _pick_inner(left: RawRelation, right: RawRelation, inner: Optional[str]) -> str:
    if inner is None:
        return "right" if len(right) <= len(left) else "left"
    if inner not in ("left", "right"):
        raise ValueError(f"inner must be 'left', 'right', or None, got {inner!r}")
    return inner


def _device(dev) -> torch.device:
    D.require_cuda()
    return torch.device("cuda", torch.cuda.current_device()) if dev is None else torch.device(dev)


def _to_matchset(m: D.DeviceMatches, left_name: str, right_name: str) -> MatchSet:
    if m.n_matches == 0:
        return MatchSet(left_name, right_name)
    lo, ro, so = m.to_host()
    return MatchSet(left_name, right_name, lo, ro, so)


def join_prepared(left: D.PreparedRelation, right: D.PreparedRelation, theta,
                  band: Optional[float] = None, left_name: str = "left",
                  right_name: str = "right") -> MatchSet:
    """Canonical MatchSet of two device-resident prepared relations."""
    t = Threshold.of(theta)
    check_dims(left.dim, right.dim)
    return _to_matchset(D.join_prepared(left, right, t.value, band), left_name, right_name)


def _run(left: RawRelation, right: RawRelation, model: EmbeddingModel, theta, threads: int,
         algo: str, inner: str, band, dev, devices=None) -> Tuple[MatchSet, JoinStats]:
    t = Threshold.of(theta)
    if threads < 1:
        raise ValueError("threads must be >= 1")
    if devices is not None and len(devices) > 1:
        return _run_devices(left, right, model, t, threads, algo, inner, band, devices)
    if devices is not None and len(devices) == 1:
        dev = devices[0]
    dev = _device(dev)
    t0 = time.perf_counter_ns()
    with torch.cuda.device(dev):
        pl = prepare_relation(model, left, dev)
        pr = prepare_relation(model, right, dev)
        m = D.join_prepared(pl, pr, t.value, band)
        matches = _to_matchset(m, left.name, right.name)
    wall = time.perf_counter_ns() - t0
    stats = JoinStats(wall_nanos=wall, model_calls_left=len(left), model_calls_right=len(right),
                      pairs_compared=len(left) * len(right), matches=len(matches),
                      peak_buffer_bytes=0, threads=threads, algo=algo, inner_relation=inner)
    return matches, stats


def copy_prepared(p: D.PreparedRelation, dev: torch.device) -> D.PreparedRelation:
    """A prepared relation copied to another device (peer copies over
    NVLink when both are GPUs of one node); bitwise the same buffers."""
    if p.device == dev:
        return p
    with torch.cuda.device(dev):
        cp = (lambda x: None if x is None else x.to(dev, non_blocking=True))
        return D.PreparedRelation(cp(p.f32), cp(p.op), p.n, p.dim, p.name, cp(p.repaired_dev),
                                  cp(p.row_err), cp(p.tile_err), cp(p.inv_norm))


def _run_devices(left: RawRelation, right: RawRelation, model: EmbeddingModel, t: Threshold,
                 threads: int, algo: str, inner: str, band, devices
                 ) -> Tuple[MatchSet, JoinStats]:
    """The operator on several GPUs of one process: the reference splits the
    outer rows over `threads` workers (join.py:121-142, row bounds
    join.py:263-264); here device k owns left rows [n*k/N, n*(k+1)/N).  The
    right relation is embedded and prepared ONCE (|S| model calls) on the
    first device and copied, prepared, to the others; every device embeds
    only its own left rows, so model calls stay |R| + |S|.  All joins are
    queued before any result is read; each device's canonical rows, shifted
    by its r0, concatenate in device order to the canonical MatchSet."""
    from .multigpu import concat_shards, shard_range
    devs = [torch.device(d) for d in devices]
    for d in devs:
        if d.type != "cuda":
            raise ValueError(f"devices must be CUDA devices, got {d}")
    D.require_cuda()
    t0 = time.perf_counter_ns()
    with torch.cuda.device(devs[0]):
        pr0 = prepare_relation(model, right, devs[0])
    pending = []
    for k, d in enumerate(devs):
        r0, r1 = shard_range(len(left), k, len(devs))
        with torch.cuda.device(d):
            pr = copy_prepared(pr0, d)
            pl = prepare_relation(model, RawRelation(left.name, left.tokens[r0:r1]), d)
            pending.append((d, D.join_prepared_async(pl, pr, t.value, band, left_base=r0)))
    parts = []
    for d, p in pending:
        with torch.cuda.device(d):
            m = p.result()
            parts.append(m.to_host() if m.n_matches else
                         (np.empty(0, np.uint64), np.empty(0, np.uint64),
                          np.empty(0, np.float32)))
    lo, ro, so = concat_shards(parts)
    matches = MatchSet(left.name, right.name, lo, ro, so) if len(lo) else \
        MatchSet(left.name, right.name)
    wall = time.perf_counter_ns() - t0
    stats = JoinStats(wall_nanos=wall, model_calls_left=len(left), model_calls_right=len(right),
                      pairs_compared=len(left) * len(right), matches=len(matches),
                      peak_buffer_bytes=0, threads=threads, algo=algo, inner_relation=inner)
    return matches, stats


def tensor_join(left: RawRelation, right: RawRelation, model: EmbeddingModel, theta,
                budget_bytes: int, threads: int = 1, *, band: Optional[float] = None,
                device=None, devices=None) -> Tuple[MatchSet, JoinStats]:
    """Tensor formulation (join.py:317-373) on the device: embed once per
    relation, normalise, fused filter + canonical recheck, canonical order.
    devices=[...] shards the left rows over several GPUs of this process
    (the reference's in-operator parallelism, join.py:121-142); the result
    is the same MatchSet."""
    Threshold.of(theta)
    if threads < 1:
        raise ValueError("threads must be >= 1")
    # the budget is validated as plan_batches does; no dense buffer exists, so
    # the tile plan itself is not built (join.py:88-108: ~6k tiles at cfg2)
    _check_budget(budget_bytes)
    return _run(left, right, model, theta, threads, "tensor", "right", band, device, devices)


def e_selection(raw: RawRelation, model: EmbeddingModel, probe: str, theta, *,
                device=None) -> Tuple[MatchSet, JoinStats]:
    """Offsets of tuples whose cosine to the embedded probe is >= theta
    (reference join.py:145-179): |R| + 1 model calls, the relation embedded
    on the device, cosines by sjb_cosine_vm (the reference's arithmetic)."""
    from .embedding import embed_relation_device
    from .linalg import cosine_vm_device
    t = Threshold.of(theta)
    dev = _device(device)
    t0 = time.perf_counter_ns()
    probe_vec = model.embed(probe)
    with torch.cuda.device(dev):
        rows = embed_relation_device(model, raw, dev)
        if len(raw):
            sims = cosine_vm_device(probe_vec, rows).cpu().numpy()
            hits = np.nonzero(sims >= np.float32(t.value))[0]
            matches = MatchSet(raw.name, "probe", hits.astype(np.uint64),
                               np.zeros(len(hits), dtype=np.uint64),
                               np.ascontiguousarray(sims[hits]))
        else:
            matches = MatchSet(raw.name, "probe")
    wall = time.perf_counter_ns() - t0
    stats = JoinStats(wall_nanos=wall, model_calls_left=len(raw), model_calls_right=1,
                      pairs_compared=len(raw), matches=len(matches), peak_buffer_bytes=0,
                      threads=1, algo="e_selection", inner_relation="right")
    return matches, stats


def nlj_prefetch(left: RawRelation, right: RawRelation, model: EmbeddingModel, theta,
                 threads: int = 1, inner: Optional[str] = None, *,
                 band: Optional[float] = None, device=None,
                 devices=None) -> Tuple[MatchSet, JoinStats]:
    """Prefetch NLJ (join.py:238-294): identical result to tensor_join; the
    inner-relation choice is recorded in the stats as the reference does."""
    inner_name = _pick_inner(left, right, inner)
    return _run(left, right, model, theta, threads, "prefetch_nlj", inner_name, band, device,
                devices)


ArrayLike = Union[np.ndarray, torch.Tensor]


def _as_device_matrix(x: ArrayLike, dev: torch.device) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        x = x.to(device=dev, dtype=torch.float32)
        return x.contiguous()
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(dev)


_STREAM_MIN_ROWS = 1 << 16   # smaller right relations: one copy, then join


def _is_host(x: ArrayLike) -> bool:
    return isinstance(x, np.ndarray) or (isinstance(x, torch.Tensor) and not x.is_cuda)


def _host_tensor(x: ArrayLike) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(torch.float32).contiguous()
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32))


def _pinned(n: int, dtype) -> torch.Tensor:
    return torch.empty(max(n, 1), dtype=dtype, pin_memory=True)


# Result bytes of the last host-input join of a shape: output-heavy joins
# (cfg5 at theta 0.4: 1.6 GB of MatchSet against a 21 ms join) are bound by
# the device->host copy of the result, which only starts once a part's join
# is done, so they split the left rows into many equal parts instead
# (cfg5 e2e 60 -> 33 ms).  Below 512 MB the three-part split wins: cfg2's
# 107 MB result, 17.4 ms e2e, took 21.6 ms in eight parts.
_result_bytes: dict = {}
HEAVY_RESULT_BYTES = 512 << 20
HEAVY_PARTS = 8


def _split_bounds(n: int, min_rows: int = 4096, heavy: bool = False):
    """Left row bounds of the host-input join: `heavy` (the shape's last
    result exceeded HEAVY_RESULT_BYTES) -> HEAVY_PARTS equal parts, so the
    result copy starts after the first eighth; else _split_bounds_light."""
    if heavy:
        step = max(min_rows, -(-n // HEAVY_PARTS)) // 1024 * 1024 or 1024
        bounds = list(range(0, n, step)) + [n]
        if len(bounds) > 2 and bounds[-1] - bounds[-2] < min_rows:
            del bounds[-2]               # fold a short tail into the last part
        return bounds
    return _split_bounds_light(n, min_rows)


def _split_bounds_light(n: int, min_rows: int = 4096):
    """Left row bounds of the host-input join: 60% of the rows in the first
    part, whose filter hides the S copy (both scale with |S|.d; the filter
    must just outlast the copy plus its last chunk), then the rest as 70% +
    30%, so the last part -- whose result copy nothing hides -- is short.
    Multiples of 1024 rows.  cfg2 e2e medians by first-part share
    (tools/e2e_split.py): 0.5 19.8 ms, 0.55 19.6, 0.58 18.5, 0.6 18.3,
    0.65 19.3.  SJB_SPLIT_FIRST overrides the share (sweeps)."""
    def r(x: float) -> int:
        return int(x) // 1024 * 1024
    h = r(n * float(os.environ.get("SJB_SPLIT_FIRST", "0.6")))
    if h < min_rows:
        return [0, n]
    m = h + r((n - h) * 0.7)
    bounds = [0, h]
    if m - h >= min_rows and n - m >= min_rows:
        bounds.append(m)
    bounds.append(n)
    return bounds


def _join_host_split(PL: D.PreparedRelation, right_host, theta: float, band,
                     left_name: str, right_name: str, ready=None,
                     heavy: bool = False, PR: Optional[D.PreparedRelation] = None,
                     sims: str = "exact") -> MatchSet:
    """Host-input join in `parts` left row ranges: the first streams S in
    (H2D overlapped with its filter); each later part is queued on the
    resident S before the previous part's count is read back, so the GPU
    never waits for the host between parts, and the previous parts' matches
    copy to pinned host memory while it runs.  All parts land in one pinned
    buffer, so the MatchSet needs no concatenation.  The ranges are disjoint
    and ordered, so the result is the canonical MatchSet (bounds:
    _split_bounds)."""
    n = PL.n
    bounds = _split_bounds(n, heavy=heavy)
    if ready is None:
        ready = lambda r: None                          # noqa: E731  (rows all prepared)
    if len(bounds) <= 2:
        ready(n)
        if PR is not None:
            m = D.join_prepared(PL, PR, theta, band, sims=sims)
        else:
            m, _ = D.join_streamed(PL, right_host, theta, band)
        return _to_matchset(m, left_name, right_name)
    dev = PL.device
    comp = torch.cuda.current_stream(dev)
    copy = torch.cuda.Stream(dev)
    ranges = list(zip(bounds[:-1], bounds[1:]))
    state = {"bufs": None, "cap": 0, "done": 0}
    keep = []

    def emit(idx: int, pending, ev) -> None:
        """Read part idx's count (later parts keep the GPU busy meanwhile)
        and queue its D2H behind its own kernels."""
        m = pending.result()
        if m.retries:                  # rerun after later parts were queued
            ev = torch.cuda.Event()
            ev.record(comp)
        k, done = m.n_matches, state["done"]
        if state["bufs"] is None or done + k > state["cap"]:
            # size from what the parts so far produced (the parts are alike)
            cap = max(int((done + k) * len(ranges) / (idx + 1) * 1.15) + 4096, done + k)
            nb = (_pinned(cap, torch.int64), _pinned(cap, torch.int64),
                  _pinned(cap, torch.float32))
            if state["bufs"] is not None:
                copy.synchronize()
                for a, o in zip(nb, state["bufs"]):
                    a[:done].copy_(o[:done])
            state["bufs"], state["cap"] = nb, cap
        copy.wait_event(ev)
        with torch.cuda.stream(copy):
            for b, d in zip(state["bufs"], (m.lefts, m.rights, m.sims)):
                b[done:done + k].copy_(d, non_blocking=True)
        keep.append(m)                                  # device columns live until copied
        state["done"] = done + k

    prev = None
    for idx, (r0, r1) in enumerate(ranges):
        ready(r1)                                       # this part's left rows, normalised
        if PR is None:
            p, PR = D.join_streamed(PL.rows(r0, r1), right_host, theta, band, sync=False)
        else:
            p = D.join_prepared_async(PL.rows(r0, r1), PR, theta, band, left_base=r0,
                                      sims=sims)
        ev = torch.cuda.Event()
        ev.record(comp)
        if prev is not None:
            emit(idx - 1, *prev)
        prev = (p, ev)
    emit(len(ranges) - 1, *prev)
    bufs, done = state["bufs"], state["done"]
    copy.synchronize()
    if done == 0:
        return MatchSet(left_name, right_name)
    return MatchSet(left_name, right_name, bufs[0][:done].numpy().view(np.uint64),
                    bufs[1][:done].numpy().view(np.uint64), bufs[2][:done].numpy())


def _is_bf16(x) -> bool:
    return isinstance(x, torch.Tensor) and x.dtype == torch.bfloat16


def tensor_join_vectors(left: ArrayLike, right: ArrayLike, theta, *,
                        band: Optional[float] = None, left_name: str = "left",
                        right_name: str = "right", device=None,
                        sims: str = "exact") -> Tuple[MatchSet, JoinStats]:
    """Join prefetched (un-normalised) vectors: the LookupModel path of the
    reference's tensor_join without the per-token dictionary.  Host or device
    inputs; host MatchSet output.

    bfloat16 tensors with dim > 128 (BASELINE cfg4) take the raw-operand
    path: the bf16 rows feed the tensor cores as they are (exact products)
    and are normalised after the GEMM, so the filter band is ~2e-4 instead
    of the 16-bit rounding band.  The result is the reference's join of the
    rows' (exact) fp32 values.  sims='tensor' (raw-operand path only)
    returns the epilogue similarity for pairs clear of the band -- within
    ~1e-6 of the canonical value -- and rechecks only the band pairs; the
    pair set is exact either way."""
    t = Threshold.of(theta)
    dev = _device(device)
    t0 = time.perf_counter_ns()
    if _is_bf16(left) and _is_bf16(right) and left.dim() == 2 and right.dim() == 2 and \
            D.kpad(left.shape[1]) > 128:
        check_dims(left.shape[1], right.shape[1])
        with torch.cuda.device(dev):
            pl = D.prepare_bf16(left.to(dev, non_blocking=True))
            pr = D.prepare_bf16(right.to(dev, non_blocking=True))
            if left.shape[0] >= HEAVY_PARTS * 4096:
                # left rows in equal parts on the resident S: each part's
                # matches copy to the host while the next part joins
                matches = _join_host_split(pl, None, t.value, band, left_name, right_name,
                                           heavy=True, PR=pr, sims=sims)
            else:
                m = D.join_prepared(pl, pr, t.value, band, sims=sims)
                matches = _to_matchset(m, left_name, right_name)
        wall = time.perf_counter_ns() - t0
        return matches, JoinStats(wall_nanos=wall, model_calls_left=left.shape[0],
                                  model_calls_right=right.shape[0],
                                  pairs_compared=left.shape[0] * right.shape[0],
                                  matches=len(matches), peak_buffer_bytes=0, threads=1,
                                  algo="tensor", inner_relation="right")
    if sims != "exact":
        raise ValueError("sims='tensor' needs bfloat16 inputs with dim > 128")
    if _is_bf16(left):
        left = left.float()                  # exact: bf16 values are fp32 values
    if _is_bf16(right):
        right = right.float()
    with torch.cuda.device(dev):
        if _is_host(right) and right.shape[0] >= _STREAM_MIN_ROWS:
            # overlap the right relation's H2D copy with the filter, and the
            # first half's result D2H with the second half's join.  Both host
            # copies are queued at once on one copy stream (left first), so
            # the link never waits for host-side setup.
            # the left rows of the first part go first, then S, then the
            # rest of the left rows (needed only by the later parts)
            comp = torch.cuda.current_stream(dev)
            copy = torch.cuda.Stream(dev)
            pieces = []
            shape_key = (left.shape[0], right.shape[0], right.shape[1], float(np.float32(t.value)))
            heavy = _result_bytes.get(shape_key, 0) > HEAVY_RESULT_BYTES
            if _is_host(left):
                lh = _host_tensor(left)
                if lh.dim() != 2:
                    raise ValueError("left must be a 2-D matrix")
                check_dims(lh.shape[1], right.shape[1])
                L = torch.empty(tuple(lh.shape), dtype=torch.float32, device=dev)
                copy.wait_stream(comp)
                b = _split_bounds(L.shape[0], heavy=heavy)
                cuts = [0, b[1], L.shape[0]] if len(b) > 2 else [0, L.shape[0]]
                spans = [(r0, r1) for r0, r1 in zip(cuts[:-1], cuts[1:]) if r1 > r0]

                def copy_rows(r0: int, r1: int) -> None:
                    D.bounce_copy(L[r0:r1], lh[r0:r1], copy)   # pinned ring if pageable
                    with torch.cuda.stream(copy):
                        ev = torch.cuda.Event()
                        ev.record(copy)
                    pieces.append((r0, r1, ev))

                if spans:
                    copy_rows(*spans[0])
            else:
                L, spans = _as_device_matrix(left, dev), []
                check_dims(L.shape[1], right.shape[1])
                pieces.append((0, L.shape[0], None))
            staged = D.stage_host(_host_tensor(right), dev, stream=copy,
                                  chunks=int(os.environ.get("SJB_STREAM_CHUNKS", "8")))
            for sp in spans[1:]:
                copy_rows(*sp)
            PL, ready = D.prepare_pieces(L, pieces)
            matches = _join_host_split(PL, staged, t.value, band, left_name, right_name,
                                       ready=ready, heavy=heavy)
            _result_bytes[shape_key] = len(matches) * 20
        else:
            L = _as_device_matrix(left, dev)
            check_dims(L.shape[1], right.shape[1])
            m = D.join_prepared(D.prepare(L), D.prepare(_as_device_matrix(right, dev)), t.value,
                                band)
            matches = _to_matchset(m, left_name, right_name)
    R = right
    wall = time.perf_counter_ns() - t0
    stats = JoinStats(wall_nanos=wall, model_calls_left=L.shape[0],
                      model_calls_right=R.shape[0], pairs_compared=L.shape[0] * R.shape[0],
                      matches=len(matches), peak_buffer_bytes=0, threads=1, algo="tensor",
                      inner_relation="right")
    return matches, stats


def join_embedded(left: EmbeddedRelation, right: EmbeddedRelation, theta, *,
                  band: Optional[float] = None, device=None) -> MatchSet:
    """Join two EmbeddedRelations; normalises them unless already normalised
    (then the rows are used as given, like tile_similarity)."""
    check_dims(left.dim, right.dim)
    t = Threshold.of(theta)
    dev = _device(device)
    with torch.cuda.device(dev):
        preps, norms = [], []
        for er in (left, right):
            x = torch.from_numpy(np.ascontiguousarray(er.data)).to(dev)
            if er.normalized:
                # re-normalising changes bits: the caller's rows are used as
                # given, cast for the filter, with a band that covers their norms
                preps.append(D.cast_prepared(x))
                norms.append(D.max_row_norm(x))
            else:
                preps.append(D.prepare(x))
                norms.append(1.0)
        if band is None and (left.normalized or right.normalized):
            band = D.band_for_rows(left.dim, *norms)
            if not np.isfinite(band):
                band = 4.0 * max(1.0, abs(float(t.value))) + 1e30
        m = D.join_prepared(preps[0], preps[1], t.value, band)
        return _to_matchset(m, left.source_name, right.source_name)
