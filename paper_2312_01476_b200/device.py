"""Device engine: prepared relations and the fused join, on torch-owned HBM.

PyTorch is used only for device memory, streams and host<->device copies;
every computation is a libsjb200.so kernel reached through the C ABI
(include/simjoin_b200.h).  There is no CPU fallback: without a CUDA device
or without the built library these functions raise.

Pipeline of one join:

  prepare(raw)         normalize_cast kernel: canonical fp32 rows (bitwise
                       sj_normalize_rows) + 16-bit operand image (tiled
                       layout; bf16 for kpad <= 128, fp16 above)
  join_prepared(L, R)  tcgen05 filter (approx >= theta - band) -> canonical
                       fp32 recheck -> row bucketing -> per-row sort ->
                       MatchSet columns (u64 lefts, u64 rights, f32 sims)

Capacity protocol (the reference's count + capacity + retry, _ckern.pyx:
165-175, 194-211): the filter writes candidates into per-CTA segments and
counts past capacity; on overflow the join is re-run once with the exact
capacity the first pass measured.  The last capacity needed for a shape is
remembered, so repeated joins of the same shape run once.
"""

from __future__ import annotations

import ctypes
import os
import threading
from dataclasses import dataclass, field
from typing import Dict, Optional, Tuple

import numpy as np
import torch

from . import _lib
from .errors import CapacityExceeded, DimensionMismatch

TILE_ROWS = 256


def _vp(t: Optional[torch.Tensor]):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def _stream(device: torch.device) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def launch_count() -> int:
    """Kernels libsjb200.so has launched in this process (all devices)."""
    return int(_lib.lib().sjb_launch_count())


def require_cuda() -> None:
    if not torch.cuda.is_available():
        raise RuntimeError("simjoin-b200 needs a CUDA device (there is no CPU fallback)")
    _lib.lib()


def kpad(dim: int) -> int:
    return int(_lib.lib().sjb_kpad(dim))


def operand_elems(n: int, dim: int) -> int:
    return int(_lib.lib().sjb_operand_elems(n, dim))


def op_dtype(dim: int) -> torch.dtype:
    """Element type of the operand image (sjb_common.cuh op_is_bf16): bf16 for
    kpad <= 128 (the resident-R filter), fp16 for the K-streaming wide path."""
    return torch.bfloat16 if kpad(dim) <= 128 else torch.float16


def op_empty(n: int, dim: int, dev: torch.device) -> torch.Tensor:
    """Uninitialised operand image for n rows (sjb_operand_elems elements)."""
    return torch.empty(operand_elems(n, dim), dtype=op_dtype(dim), device=dev)


def default_band(dim: int) -> float:
    """Provably sufficient 16-bit filter margin for unit vectors (C ABI
    sjb_default_band): 2e + e^2 + accumulation slack, e = u + 2^-25 sqrt(d),
    u = 2^-8 for bf16 operands (kpad <= 128), 2^-11 for fp16 (above)."""
    return float(_lib.lib().sjb_default_band(dim))


@dataclass
class PreparedRelation:
    """A relation resident in HBM in the two forms the join reads."""

    f32: torch.Tensor          # (n, dim) canonical normalised fp32 rows
    op: torch.Tensor           # 16-bit operand image (op_dtype; sjb_operand_elems elements)
    n: int
    dim: int
    name: str = ""
    repaired_dev: Optional[torch.Tensor] = None  # (1,) int64 repaired-row counter
    # 16-bit rounding errors (sjb_join_args.left_row_err / right_tile_err):
    row_err: Optional[torch.Tensor] = None       # (n,) >= ||op(x_i) - x_i||
    tile_err: Optional[torch.Tensor] = None      # (tiles,) max over each 256-row tile
    # raw-operand relations (prepare_bf16): op holds the raw bf16 rows and
    # inv_norm[i] = RN(1 / ||x_i||) (rows padded to 512, 0 past n)
    inv_norm: Optional[torch.Tensor] = None

    @property
    def device(self) -> torch.device:
        return self.f32.device

    def repaired(self) -> int:
        return int(self.repaired_dev.item()) if self.repaired_dev is not None else 0

    def rows(self, r0: int, r1: int) -> "PreparedRelation":
        """Rows [r0, r1) as a prepared relation (views, no copy); r0 must sit
        on a 512-row boundary (an operand tile pair)."""
        if r0 % (2 * TILE_ROWS) or not 0 <= r0 <= r1 <= self.n:
            raise ValueError(f"bad row range [{r0}, {r1}) of {self.n}")
        kp = kpad(self.dim)
        t0 = r0 // TILE_ROWS
        return PreparedRelation(self.f32[r0:r1], self.op[t0 * TILE_ROWS * kp:], r1 - r0,
                                self.dim, self.name, None,
                                None if self.row_err is None else self.row_err[r0:r1],
                                None if self.tile_err is None else self.tile_err[t0:],
                                None if self.inv_norm is None else self.inv_norm[r0:])

    @property
    def raw(self) -> bool:
        return self.inv_norm is not None


def tile_count(n: int) -> int:
    return int(_lib.lib().sjb_tile_count(n))


def _err_buffers(n: int, dev: torch.device) -> Tuple[torch.Tensor, torch.Tensor]:
    return (torch.empty(max(n, 1), dtype=torch.float32, device=dev),
            torch.empty(max(tile_count(n), 1), dtype=torch.float32, device=dev))


def _check_matrix(x: torch.Tensor, what: str) -> None:
    if not x.is_cuda:
        raise ValueError(f"{what} must be a CUDA tensor")
    if x.dtype != torch.float32 or x.dim() != 2:
        raise ValueError(f"{what} must be a 2-D float32 tensor, got {x.dtype} {tuple(x.shape)}")
    if not x.is_contiguous():
        raise ValueError(f"{what} must be row-major contiguous")


def prepare(raw: torch.Tensor, name: str = "", out32: Optional[torch.Tensor] = None
            ) -> PreparedRelation:
    """Normalise rows (bitwise sj_normalize_rows) and build the operand image."""
    _check_matrix(raw, "relation")
    L = _lib.lib()
    n, dim = raw.shape
    dev = raw.device
    f32 = out32 if out32 is not None else torch.empty_like(raw)
    op = op_empty(n, dim, dev)
    rep = torch.zeros(1, dtype=torch.int64, device=dev)
    re, te = _err_buffers(n, dev)
    with torch.cuda.device(dev):
        _lib.check(L.sjb_normalize_rows(_vp(raw), n, dim, _vp(f32), _vp(op), _vp(rep), _vp(re),
                                        _vp(te), _stream(dev)), "sjb_normalize_rows")
    return PreparedRelation(f32, op, n, dim, name, rep, re, te)


def raw_band(dim: int) -> float:
    """Filter band of raw-operand (bf16) joins (C ABI sjb_raw_band): exact
    products, so only accumulation and the normalisation roundings."""
    return float(_lib.lib().sjb_raw_band(dim))


def prepare_bf16(raw: torch.Tensor, name: str = "") -> PreparedRelation:
    """A bf16 relation (n, dim > 128) for the raw-operand wide filter
    (sjb_prepare_bf16): canonical normalised fp32 rows (bitwise the
    reference's normalize_rows of the rows' exact fp32 values), the RAW bf16
    rows as the operand image, and the rows' inverse norms."""
    if not raw.is_cuda or raw.dtype != torch.bfloat16 or raw.dim() != 2:
        raise ValueError("prepare_bf16 needs a 2-D bfloat16 CUDA tensor")
    raw = raw.contiguous()
    n, dim = raw.shape
    if kpad(dim) <= 128:
        raise ValueError("raw-operand relations are for dim > 128 (the wide filter)")
    dev = raw.device
    f32 = torch.empty((n, dim), dtype=torch.float32, device=dev)
    op = torch.empty(operand_elems(n, dim), dtype=torch.bfloat16, device=dev)
    inv = torch.empty(max(operand_elems(n, dim) // kpad(dim), 1), dtype=torch.float32, device=dev)
    rep = torch.zeros(1, dtype=torch.int64, device=dev)
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().sjb_prepare_bf16(_vp(raw), n, dim, _vp(f32), _vp(op), _vp(inv),
                                               _vp(rep), _stream(dev)), "sjb_prepare_bf16")
    return PreparedRelation(f32, op, n, dim, name, rep, None, None, inv)


def _raw_mode(L: PreparedRelation, R: PreparedRelation) -> bool:
    if L.raw != R.raw:
        raise ValueError("both relations must be raw-operand (prepare_bf16) or neither")
    return L.raw


SIMS_MODES = {"exact": 0, "tensor": 1}


def _sims_mode(sims: str, raw: bool) -> int:
    if sims not in SIMS_MODES:
        raise ValueError(f"sims must be one of {sorted(SIMS_MODES)}, got {sims!r}")
    if sims == "tensor" and not raw:
        raise ValueError("sims='tensor' needs raw-operand (bf16, dim > 128) relations")
    return SIMS_MODES[sims]


def prepare_pieces(raw: torch.Tensor, pieces, name: str = ""):
    """prepare() for a device matrix whose rows land in pieces: `pieces` is
    [(r0, r1, event)] in row order, r0 on 512-row boundaries, each piece
    complete when its event fires (None: already there).  Returns the
    PreparedRelation and ready(r): queue, on the current stream, the wait and
    normalisation of every piece starting below row r not yet done -- so a
    join of the first rows can start before the later rows have arrived."""
    _check_matrix(raw, "relation")
    lib = _lib.lib()
    n, dim = raw.shape
    dev = raw.device
    f32 = torch.empty_like(raw)
    op = op_empty(n, dim, dev)
    rep = torch.zeros(1, dtype=torch.int64, device=dev)
    re, te = _err_buffers(n, dev)
    kp = kpad(dim)
    todo = list(pieces)

    def ready(r: int) -> None:
        with torch.cuda.device(dev):
            while todo and todo[0][0] < r:
                r0, r1, ev = todo.pop(0)
                if ev is not None:
                    torch.cuda.current_stream(dev).wait_event(ev)
                t0 = r0 // TILE_ROWS
                _lib.check(lib.sjb_normalize_rows(
                    ctypes.c_void_p(raw.data_ptr() + r0 * dim * 4), r1 - r0, dim,
                    ctypes.c_void_p(f32.data_ptr() + r0 * dim * 4),
                    ctypes.c_void_p(op.data_ptr() + t0 * TILE_ROWS * kp * 2), _vp(rep),
                    ctypes.c_void_p(re.data_ptr() + r0 * 4),
                    ctypes.c_void_p(te.data_ptr() + t0 * 4), _stream(dev)),
                    "sjb_normalize_rows")

    return PreparedRelation(f32, op, n, dim, name, rep, re, te), ready


def cast_prepared(rows: torch.Tensor, name: str = "") -> PreparedRelation:
    """Rows used AS GIVEN (already normalised by the caller): the fp32 rows
    are the caller's tensor and the operand image is their 16-bit cast
    (sjb_cast_rows).  No rounding errors are recorded, so joins of such a
    relation filter with a uniform band -- which must cover the rows' norms
    (band_for_rows)."""
    _check_matrix(rows, "relation")
    n, dim = rows.shape
    dev = rows.device
    op = op_empty(n, dim, dev)
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().sjb_cast_rows(_vp(rows), n, dim, _vp(op), _stream(dev)),
                   "sjb_cast_rows")
    return PreparedRelation(rows, op, n, dim, name, None, None, None)


def max_row_norm(rows: torch.Tensor) -> float:
    """Largest row norm (fp64 sums, sjb_row_norms), rounded up slightly."""
    n, dim = rows.shape
    if n == 0:
        return 0.0
    out = torch.empty(n, dtype=torch.float32, device=rows.device)
    with torch.cuda.device(rows.device):
        _lib.check(_lib.lib().sjb_row_norms(_vp(rows), n, dim, _vp(out), _stream(rows.device)),
                   "sjb_row_norms")
    m = float(out.max().item())
    return m * (1 + 1e-6) if np.isfinite(m) else float("inf")


def band_for_rows(dim: int, max_norm_left: float, max_norm_right: float) -> float:
    """Filter band for rows of norm <= M (not necessarily unit): each
    operand error grows at most like the norm (||op(x) - x|| <= M e when
    M >= 1), so |approx - exact| <= M_L M_R (2e + e^2) and the fp32
    accumulation slack scales with ||op(x)|| ||op(y)|| <= M_L M_R (1 + e)^2:
    the unit-row band (sjb_default_band) times max(1, M_L) max(1, M_R) and
    1.01 (covers the (1 + e)^2 factor).  Non-finite norms give an infinite
    band: every pair is rechecked canonically."""
    ml, mr = max(1.0, max_norm_left), max(1.0, max_norm_right)
    if not (np.isfinite(ml) and np.isfinite(mr)):
        return float("inf")
    return default_band(dim) * ml * mr * 1.01


def normalize_rows_(m: torch.Tensor) -> torch.Tensor:
    """In-place fp32 row normalisation; returns the (1,) int64 repaired count."""
    _check_matrix(m, "matrix")
    rep = torch.zeros(1, dtype=torch.int64, device=m.device)
    with torch.cuda.device(m.device):
        _lib.check(_lib.lib().sjb_normalize_rows(_vp(m), m.shape[0], m.shape[1], _vp(m),
                                                 ctypes.c_void_p(0), _vp(rep), None, None,
                                                 _stream(m.device)), "sjb_normalize_rows")
    return rep


@dataclass
class DeviceMatches:
    """Canonical match columns on the device (int64 tensors hold u64 values)."""

    lefts: torch.Tensor
    rights: torch.Tensor
    sims: torch.Tensor
    n_matches: int
    n_candidates: int
    cand_capacity: int
    retries: int
    grid: int

    def to_host(self) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
        """Copy the columns into pinned host memory (torch's caching host
        allocator, so repeated joins reuse the pinned blocks) and return
        numpy views that own them."""
        outs = []
        for t in (self.lefts, self.rights, self.sims):
            h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
            h.copy_(t, non_blocking=True)
            outs.append(h)
        torch.cuda.current_stream(self.lefts.device).synchronize()
        return (outs[0].numpy().view(np.uint64), outs[1].numpy().view(np.uint64),
                outs[2].numpy())


_cap_lock = threading.Lock()
_cap_cache: Dict[tuple, int] = {}

# Recheck placement (sjb_join_args.recheck): joins whose last run of the same
# shape had more candidates than this fraction of the pairs recheck in a
# full-occupancy kernel after the filter; sparser ones inside it.
DENSE_FRACTION = 2e-4


def _recheck_mode(key: tuple, pairs: int) -> int:
    with _cap_lock:
        seen = _cap_cache.get(key, 0)
    return 1 if pairs > 0 and seen > DENSE_FRACTION * pairs else 0

# workspace is cached per (device, host thread) and grown on demand: joins
# issued concurrently from several host threads (the reference runs kernel
# backends from `threads` workers, join.py:121-142) must not share counters
_ws_cache: Dict[tuple, torch.Tensor] = {}


def _ws_key(dev: torch.device) -> tuple:
    idx = dev.index if dev.index is not None else torch.cuda.current_device()
    return idx, threading.get_ident()


def _workspace(nbytes: int, dev: torch.device) -> torch.Tensor:
    key = _ws_key(dev)
    with _cap_lock:
        ws = _ws_cache.get(key)
    if ws is None or ws.numel() < nbytes:
        ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=dev)
        with _cap_lock:
            _ws_cache[key] = ws
    return ws


def _ws_bytes_cached(dev: torch.device) -> int:
    with _cap_lock:
        ws = _ws_cache.get(_ws_key(dev))
    return 0 if ws is None else ws.numel()


def release_workspaces() -> None:
    _ws_cache.clear()


def initial_capacity(n_left: int, n_right: int) -> int:
    """First-try candidate capacity when nothing is known about selectivity."""
    pairs = n_left * n_right
    return int(max(1 << 20, min(pairs, 1 << 24)))


# Cold joins (no capacity history for the shape) above this many pairs size
# their candidate buffers from a sampled pre-pass instead of the fixed first
# guess, so a selective-but-dense join (cfg5 at theta 0.4: 8.1e7 candidates)
# does not run twice; smaller joins retry cheaply if they overflow.
PREPASS_MIN_PAIRS = 2_000_000_000
PREPASS_ROWS = 2048


def _prepass_capacity(L: PreparedRelation, R: PreparedRelation, theta: float, band,
                      per_row_band: bool, sims: str) -> int:
    """Candidates of a contiguous 2048-row sample of the left relation (from
    its middle, on a 512-row boundary) joined with all of R, scaled to all
    of L, plus 20% and 64k slack: the first call's capacity.  The sample's
    own capacity is the fixed first guess (it retries if that overflows)."""
    rows = min(L.n, PREPASS_ROWS)
    r0 = ((L.n - rows) // 2) // (2 * TILE_ROWS) * (2 * TILE_ROWS)
    sample = L.rows(r0, r0 + rows)
    m = join_prepared(sample, R, theta, band, cand_cap=initial_capacity(rows, R.n),
                      per_row_band=per_row_band, sims=sims)
    est = m.n_candidates * (L.n / max(rows, 1))
    return int(est * 1.2) + (1 << 16)


class PendingJoin:
    """A join whose kernels are queued but whose match count (data dependent)
    has not been read back yet.  result() blocks on that count, reruns the
    join with the exact capacity if the candidate segments overflowed, and
    returns the DeviceMatches; later work can be queued before calling it."""

    def __init__(self, info_t: torch.Tensor, finish):
        # the 40-byte info copy is queued now, right behind the join, and
        # waited on through an event: a later .cpu() would also wait for
        # everything queued after the join on the stream
        with torch.cuda.device(info_t.device):
            self._info_h = torch.empty(info_t.shape, dtype=info_t.dtype, pin_memory=True)
            self._info_h.copy_(info_t, non_blocking=True)
            self._ev = torch.cuda.Event()
            self._ev.record(torch.cuda.current_stream(info_t.device))
        self._finish, self._done = finish, None

    def result(self) -> "DeviceMatches":
        if self._done is None:
            self._ev.synchronize()
            self._done = self._finish(self._info_h.numpy())
        return self._done


def join_prepared(L: PreparedRelation, R: PreparedRelation, theta: float,
                  band: Optional[float] = None, cand_cap: Optional[int] = None,
                  left_base: int = 0, grid: int = 0, tiles_per_chunk: int = 0,
                  max_bytes: Optional[int] = None,
                  filter_events: Optional[Tuple[torch.cuda.Event, torch.cuda.Event]] = None,
                  per_row_band: bool = True, sims: str = "exact") -> DeviceMatches:
    """Canonical threshold join of two prepared relations (device-resident).

    Blocks once at the end to read the match count (the output size is data
    dependent); everything else is asynchronous on the current stream.
    per_row_band: when both relations carry their fp16 rounding errors, filter
    with the per-row band (never looser than `band`; same result, fewer
    candidates to recheck).
    """
    return join_prepared_async(L, R, theta, band, cand_cap, left_base, grid, tiles_per_chunk,
                               max_bytes, filter_events, per_row_band, sims=sims).result()


def join_prepared_async(L: PreparedRelation, R: PreparedRelation, theta: float,
                        band: Optional[float] = None, cand_cap: Optional[int] = None,
                        left_base: int = 0, grid: int = 0, tiles_per_chunk: int = 0,
                        max_bytes: Optional[int] = None,
                        filter_events: Optional[Tuple[torch.cuda.Event, torch.cuda.Event]] = None,
                        per_row_band: bool = True, _retries: int = 0,
                        sims: str = "exact") -> PendingJoin:
    """join_prepared without the final read-back: the kernels are queued on
    the current stream and a PendingJoin is returned.  Raw-operand (bf16)
    relations filter with raw_band; sims='tensor' then emits the epilogue
    similarity for pairs clear of the band (the pair set stays exact)."""
    if L.dim != R.dim:
        raise DimensionMismatch(f"dimension mismatch: {L.dim} vs {R.dim}")
    if L.device != R.device:
        raise ValueError("relations live on different devices")
    lib = _lib.lib()
    dev = L.device
    raw = _raw_mode(L, R)
    smode = _sims_mode(sims, raw)
    theta32 = float(np.float32(theta))
    band = (raw_band(L.dim) if raw else default_band(L.dim)) if band is None else float(band)
    use_err = per_row_band and not raw and L.row_err is not None and R.tile_err is not None
    key = (L.n, R.n, L.dim, theta32, float(np.float32(band)), grid, tiles_per_chunk, use_err,
           raw, smode)
    if cand_cap is None:
        with _cap_lock:
            known = _cap_cache.get(key, 0)
        if known == 0 and L.n * R.n >= PREPASS_MIN_PAIRS and L.n >= 2 * PREPASS_ROWS:
            known = _prepass_capacity(L, R, theta, band, per_row_band, sims)
            with _cap_lock:               # also picks the recheck placement below
                _cap_cache[key] = max(_cap_cache.get(key, 0), known)
        cand_cap = max(known, initial_capacity(L.n, R.n))
    ev0 = ev1 = None
    if filter_events is not None:
        for e in filter_events:
            if not e.cuda_event:       # torch creates the CUevent on first record
                e.record(torch.cuda.current_stream(dev))
        ev0 = ctypes.c_void_p(filter_events[0].cuda_event)
        ev1 = ctypes.c_void_p(filter_events[1].cuda_event)
    with torch.cuda.device(dev):
        stream = _stream(dev)
        args = _lib.JoinArgs(n_left=L.n, n_right=R.n, dim=L.dim, theta=theta32, band=band,
                             cand_cap=int(cand_cap), out_cap=int(cand_cap),
                             left_base=int(left_base), grid=int(grid),
                             tiles_per_chunk=int(tiles_per_chunk),
                             ev_filter_begin=ev0, ev_filter_end=ev1,
                             left_row_err=L.row_err.data_ptr() if use_err else None,
                             right_tile_err=R.tile_err.data_ptr() if use_err else None,
                             recheck=_recheck_mode(key, L.n * R.n),
                             left_inv_norm=L.inv_norm.data_ptr() if raw else None,
                             right_inv_norm=R.inv_norm.data_ptr() if raw else None,
                             sims_mode=smode)
        ws_bytes = int(lib.sjb_join_workspace_bytes(ctypes.byref(args)))
        if ws_bytes < 0:
            _lib.check(-3, "sjb_join_workspace_bytes")
        out_bytes = int(cand_cap) * 20
        if _retries and max_bytes is None:
            free, _total = torch.cuda.mem_get_info(dev)
            max_bytes = int(free * 0.8) + _ws_bytes_cached(dev)
        if max_bytes is not None and ws_bytes + out_bytes > max_bytes:
            raise CapacityExceeded(
                f"join needs {ws_bytes + out_bytes} B of device memory for "
                f"{cand_cap} candidates; {max_bytes} B available")
        ws = _workspace(ws_bytes, dev)
        lefts = torch.empty(max(int(cand_cap), 1), dtype=torch.int64, device=dev)
        rights = torch.empty_like(lefts)
        sims_out = torch.empty(max(int(cand_cap), 1), dtype=torch.float32, device=dev)
        info_t = torch.zeros(5, dtype=torch.int64, device=dev)
        _lib.check(lib.sjb_join_prepared_async(
            _vp(L.f32), _vp(L.op), _vp(R.f32), _vp(R.op), ctypes.byref(args), _vp(ws),
            ws_bytes, _vp(lefts), _vp(rights), _vp(sims_out), _vp(info_t), stream),
            "sjb_join_prepared_async")

    def finish(info) -> DeviceMatches:
        n_matches, n_cand, needed = int(info[0]), int(info[1]), int(info[2])
        flags = info[3:4].view(np.int32)
        overflow, used_grid = int(flags[0]), int(flags[1])
        if overflow:
            if _retries >= 2:
                raise CapacityExceeded(f"candidate capacity still overflows after {_retries} "
                                       f"retries (needed {needed})")
            with torch.cuda.device(dev):
                return join_prepared_async(
                    L, R, theta, band, max(needed, n_matches, int(cand_cap) + 1), left_base, grid,
                    tiles_per_chunk, max_bytes, filter_events, per_row_band,
                    _retries + 1, sims=sims).result()
        with _cap_lock:
            _cap_cache[key] = max(_cap_cache.get(key, 0), needed)
        return DeviceMatches(lefts[:n_matches], rights[:n_matches], sims_out[:n_matches], n_matches,
                             n_cand, int(cand_cap), _retries, used_grid)

    return PendingJoin(info_t, finish)


def _join_args(L: PreparedRelation, n_right: int, theta32: float, band: float, cand_cap: int,
               left_base: int, use_err: bool, right_tile_err: Optional[torch.Tensor],
               recheck: int = 0, grid: int = 0, right_inv: Optional[torch.Tensor] = None,
               sims_mode: int = 0) -> "_lib.JoinArgs":
    return _lib.JoinArgs(n_left=L.n, n_right=n_right, dim=L.dim, theta=theta32, band=band,
                         cand_cap=int(cand_cap), out_cap=int(cand_cap), left_base=int(left_base),
                         grid=int(grid), tiles_per_chunk=0, ev_filter_begin=None, ev_filter_end=None,
                         left_row_err=L.row_err.data_ptr() if use_err else None,
                         right_tile_err=right_tile_err.data_ptr() if use_err else None,
                         recheck=recheck,
                         left_inv_norm=L.inv_norm.data_ptr() if right_inv is not None else None,
                         right_inv_norm=right_inv.data_ptr() if right_inv is not None else None,
                         sims_mode=sims_mode)


def _stream_chunks(n: int, chunks: int, lead: int = 4):
    """Row ranges on 512-row boundaries (operand tile pairs): a short first
    chunk (1/lead of a regular one) so the filter starts early, then ~n/chunks
    rows each."""
    step = max(512, -(-n // max(chunks, 1)) // 512 * 512 or 512)
    first = max(512, step // max(lead, 1) // 512 * 512)
    spans, r0 = [], 0
    if n > step:
        spans.append((0, min(n, first)))
        r0 = spans[-1][1]
    while r0 < n:
        spans.append((r0, min(n, r0 + step)))
        r0 += step
    return spans


class JoinSession:
    """One join whose right relation becomes ready in row ranges (the C ABI's
    incremental join: sjb_join_begin, sjb_join_filter_tiles per range,
    sjb_join_finish).  `R` is the PreparedRelation the rows are prepared
    into; filter_rows(r0, r1) queues the filter + recheck of rows [r0, r1)
    (ranges disjoint, in order, r0 on 256-row tile boundaries) once those rows
    are prepared on the current stream; finish() queues the canonical-order
    pass and returns a PendingJoin.  On candidate overflow the PendingJoin
    reruns the whole join on R (complete by then) with the measured capacity.
    `grid` < SM count leaves SMs free for kernels that must run beside the
    filter (NCCL's collective kernels in the multi-GPU streamed join)."""

    def __init__(self, L: PreparedRelation, R: PreparedRelation, theta: float,
                 band: Optional[float] = None, left_base: int = 0, grid: int = 0,
                 sims: str = "exact"):
        if L.dim != R.dim:
            raise DimensionMismatch(f"dimension mismatch: {L.dim} vs {R.dim}")
        self.L, self.R, self.theta, self.left_base, self.grid = L, R, theta, left_base, grid
        self.sims = sims
        self.lib = _lib.lib()
        dev = self.dev = L.device
        n, dim = R.n, R.dim
        raw = _raw_mode(L, R)
        smode = _sims_mode(sims, raw)
        theta32 = float(np.float32(theta))
        self.band = band = ((raw_band(dim) if raw else default_band(dim)) if band is None
                            else float(band))
        self.key = (L.n, n, dim, theta32, float(np.float32(band)), grid, 0, not raw, raw, smode)
        with _cap_lock:
            self.cand_cap = max(_cap_cache.get(self.key, 0), initial_capacity(L.n, n))
        self.empty = L.n == 0 or n == 0
        if self.empty:
            return
        use_err = not raw and L.row_err is not None and R.tile_err is not None
        with torch.cuda.device(dev):
            self.args = _join_args(L, n, theta32, band, self.cand_cap, left_base, use_err,
                                   R.tile_err, _recheck_mode(self.key, L.n * n), grid,
                                   R.inv_norm if raw else None, smode)
            self.ws_bytes = int(self.lib.sjb_join_workspace_bytes(ctypes.byref(self.args)))
            if self.ws_bytes < 0:
                _lib.check(-3, "sjb_join_workspace_bytes")
            self.ws = _workspace(self.ws_bytes, dev)
            cap = max(int(self.cand_cap), 1)
            self.lefts = torch.empty(cap, dtype=torch.int64, device=dev)
            self.rights = torch.empty_like(self.lefts)
            self.sims_out = torch.empty(cap, dtype=torch.float32, device=dev)
            self.info_t = torch.zeros(5, dtype=torch.int64, device=dev)
            _lib.check(self.lib.sjb_join_begin(ctypes.byref(self.args), _vp(self.ws),
                                               self.ws_bytes, _stream(dev)), "sjb_join_begin")

    def filter_rows(self, r0: int, r1: int, launch_grid: int = 0) -> None:
        """Filter rows [r0, r1) of R; launch_grid > 0 launches the (dim <=
        128) filter on that many CTAs only (SMs left for NCCL)."""
        if self.empty or r1 <= r0:
            return
        if r0 % TILE_ROWS:
            raise ValueError(f"row range [{r0}, {r1}) does not start on a tile boundary")
        L, R = self.L, self.R
        self.args.launch_grid = int(launch_grid)
        with torch.cuda.device(self.dev):
            _lib.check(self.lib.sjb_join_filter_tiles(
                _vp(L.f32), _vp(L.op), _vp(R.f32), _vp(R.op), ctypes.byref(self.args),
                _vp(self.ws), self.ws_bytes, r0 // TILE_ROWS, -(-min(r1, R.n) // TILE_ROWS),
                _stream(self.dev)), "sjb_join_filter_tiles")

    def finish(self) -> PendingJoin:
        L, R, dev = self.L, self.R, self.dev
        if self.empty:
            return join_prepared_async(L, R, self.theta, self.band, left_base=self.left_base,
                                       sims=self.sims)
        with torch.cuda.device(dev):
            _lib.check(self.lib.sjb_join_finish(
                _vp(L.f32), _vp(R.f32), ctypes.byref(self.args), _vp(self.ws), self.ws_bytes,
                _vp(self.lefts), _vp(self.rights), _vp(self.sims_out), _vp(self.info_t),
                _stream(dev)), "sjb_join_finish")
        cand_cap, key = self.cand_cap, self.key

        def finish(info) -> DeviceMatches:
            n_matches, n_cand, needed = int(info[0]), int(info[1]), int(info[2])
            flags = info[3:4].view(np.int32)
            if int(flags[0]):
                # candidate capacity overflowed: R is complete now; rerun with room
                with torch.cuda.device(dev):
                    m = join_prepared(L, R, self.theta, self.band,
                                      cand_cap=max(needed, n_matches, cand_cap + 1),
                                      left_base=self.left_base, grid=self.grid, sims=self.sims)
                m.retries += 1
                return m
            with _cap_lock:
                _cap_cache[key] = max(_cap_cache.get(key, 0), needed)
            return DeviceMatches(self.lefts[:n_matches], self.rights[:n_matches],
                                 self.sims_out[:n_matches], n_matches, n_cand, int(cand_cap), 0,
                                 int(flags[1]))

        return PendingJoin(self.info_t, finish)


def empty_prepared(n: int, dim: int, dev: torch.device, name: str = "",
                   rows: Optional[int] = None, f32: Optional[torch.Tensor] = None
                   ) -> PreparedRelation:
    """Uninitialised prepared buffers for a relation of n rows whose rows are
    prepared later (piece by piece, or by another rank and gathered).  `rows`
    >= n over-allocates every buffer to `rows` rows (a multiple of 512) so
    equal-sized pieces tile it; only the first n rows are joined."""
    rows = n if rows is None else rows
    if f32 is None:
        f32 = torch.empty((rows, dim), dtype=torch.float32, device=dev)
    rep = torch.zeros(1, dtype=torch.int64, device=dev)
    re, te = _err_buffers(rows, dev)
    return PreparedRelation(f32, op_empty(rows, dim, dev), n, dim, name, rep, re, te)


def prepare_into(raw: torch.Tensor, R: PreparedRelation, r0: int) -> None:
    """Normalise raw rows (m, dim) into rows [r0, r0 + m) of the prepared
    buffers R (r0 on a 512-row boundary), on the current stream."""
    _check_matrix(raw, "relation")
    m, dim = raw.shape
    if r0 % (2 * TILE_ROWS) or dim != R.dim or r0 + m > R.f32.shape[0]:
        raise ValueError(f"bad piece [{r0}, {r0 + m}) for prepared rows {R.f32.shape[0]}")
    if m == 0:
        return
    kp = kpad(dim)
    t0 = r0 // TILE_ROWS
    with torch.cuda.device(R.device):
        _lib.check(_lib.lib().sjb_normalize_rows(
            _vp(raw), m, dim, ctypes.c_void_p(R.f32.data_ptr() + r0 * dim * 4),
            ctypes.c_void_p(R.op.data_ptr() + t0 * TILE_ROWS * kp * 2), _vp(R.repaired_dev),
            ctypes.c_void_p(R.row_err.data_ptr() + r0 * 4),
            ctypes.c_void_p(R.tile_err.data_ptr() + t0 * 4), _stream(R.device)),
            "sjb_normalize_rows")


def join_chunked(L: PreparedRelation, raw: torch.Tensor, arrive, theta: float,
                 band: Optional[float] = None, left_base: int = 0, chunks: int = 8,
                 inplace: bool = False, name: str = "", spans=None, sync: bool = True,
                 grid: int = 0) -> Tuple["DeviceMatches", PreparedRelation]:
    """Join a prepared left relation with a right relation that becomes
    available on the device chunk by chunk.

    `raw` is the (n, dim) device buffer the right rows land in; arrive(r0, r1)
    must make rows [r0, r1) of it ready on the current stream (wait for a
    copy or a broadcast) -- it is called in row order, on 512-row boundaries.
    Each chunk is then normalised (canonical fp32 rows + its tiles of the
    operand image + rounding errors; in place when `inplace`) and its S tiles
    are filtered at once (JoinSession), so the filter overlaps the arrival of
    later chunks.  Same result as prepare + join_prepared.  Returns the
    matches (a PendingJoin when sync=False) and the prepared right relation
    (resident, reusable: every span is normalised even when L is empty)."""
    dev = L.device
    n, dim = raw.shape
    if dim != L.dim:
        raise DimensionMismatch(f"dimension mismatch: {L.dim} vs {dim}")
    R = empty_prepared(n, dim, dev, name, f32=raw if inplace else None)
    spans = _stream_chunks(n, chunks) if spans is None else spans
    session = JoinSession(L, R, theta, band, left_base, grid)
    with torch.cuda.device(dev):
        for r0, r1 in spans:
            arrive(r0, r1)
            prepare_into(raw[r0:r1], R, r0)
            session.filter_rows(r0, r1)
        pending = session.finish()
    return (pending if not sync else pending.result()), R


class _Bounce:
    """Pinned staging ring for PAGEABLE host -> device copies.  A pageable
    cudaMemcpy is staged by the driver one buffer at a time (~9 GB/s here);
    instead several host threads fill a pinned slot (numpy copies release
    the GIL) while the copy engine drains the previous slot.  Slots are
    reused once their copy's event has fired."""

    SLOT_BYTES = int(os.environ.get("SJB_BOUNCE_SLOT_MB", "16")) << 20
    N_SLOTS = int(os.environ.get("SJB_BOUNCE_SLOTS", "4"))
    THREADS = int(os.environ.get("SJB_BOUNCE_THREADS", "4"))

    def __init__(self):
        from concurrent.futures import ThreadPoolExecutor
        self.slots = [torch.empty(self.SLOT_BYTES, dtype=torch.uint8, pin_memory=True)
                      for _ in range(self.N_SLOTS)]
        self.views = [t.numpy() for t in self.slots]
        self.events: list = [None] * self.N_SLOTS
        self.k = 0
        self.pool = ThreadPoolExecutor(self.THREADS)
        self.lock = threading.Lock()

    def copy(self, dst: torch.Tensor, src: np.ndarray, stream: torch.cuda.Stream) -> None:
        """Queue dst <- src (same byte size; dst a contiguous CUDA tensor) on
        `stream`; returns once the last slot has been filled."""
        sb = np.ascontiguousarray(src).reshape(-1).view(np.uint8)
        db = dst.reshape(-1).view(torch.uint8)
        if sb.size != db.numel():
            raise ValueError("bounce copy: size mismatch")
        with self.lock:
            for off in range(0, sb.size, self.SLOT_BYTES):
                n = min(self.SLOT_BYTES, sb.size - off)
                i = self.k % self.N_SLOTS
                self.k += 1
                if self.events[i] is not None:
                    self.events[i].synchronize()
                per = -(-n // self.THREADS)
                step = -(-per // 4096) * 4096
                futs = [self.pool.submit(np.copyto, self.views[i][a:min(n, a + step)],
                                         sb[off + a:off + min(n, a + step)])
                        for a in range(0, n, step)]
                for f in futs:
                    f.result()
                with torch.cuda.stream(stream):
                    db[off:off + n].copy_(self.slots[i][:n], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(stream)
                self.events[i] = ev


_bounce: Optional[_Bounce] = None


def bounce_copy(dst: torch.Tensor, src: torch.Tensor, stream: torch.cuda.Stream) -> None:
    """dst (CUDA) <- src (host): pinned sources copy directly (async); pageable
    ones go through the pinned staging ring (_Bounce)."""
    global _bounce
    if src.is_pinned():
        with torch.cuda.stream(stream):
            dst.copy_(src, non_blocking=True)
        return
    with _cap_lock:
        if _bounce is None:
            _bounce = _Bounce()
    _bounce.copy(dst, src.numpy(), stream)


class StagedCopy:
    """A host matrix copied to the device in row chunks on a side stream
    (`stage_host`): `raw` is the device buffer and chunk k covers rows
    spans[k].  From pinned memory every chunk copy is queued at once; from
    pageable memory each is issued when the join reaches it (a pageable copy
    blocks the host, which then overlaps the filter of the previous chunk)."""

    def __init__(self, src: torch.Tensor, raw: torch.Tensor, spans, stream: torch.cuda.Stream,
                 eager: bool):
        self.src, self.raw, self.spans, self.stream = src, raw, spans, stream
        self.events = [None] * len(spans)
        if eager:
            for k in range(len(spans)):
                self._issue(k)

    def _issue(self, k: int) -> None:
        r0, r1 = self.spans[k]
        bounce_copy(self.raw[r0:r1], self.src[r0:r1], self.stream)
        with torch.cuda.stream(self.stream):
            ev = torch.cuda.Event()
            ev.record(self.stream)
        self.events[k] = ev

    def arrive(self, r0: int, r1: int) -> None:
        """Make rows [r0, r1) (a span) ready on the current stream."""
        k = self.spans.index((r0, r1))
        if self.events[k] is None:
            self._issue(k)
        torch.cuda.current_stream(self.raw.device).wait_event(self.events[k])


def stage_host(src: torch.Tensor, dev: torch.device, chunks: int = 8,
               stream: Optional[torch.cuda.Stream] = None) -> StagedCopy:
    """Start the chunked H2D copy of a host float32 matrix on a copy stream,
    so the link is busy from the start of a join instead of from its first
    filter launch (pinned sources: all chunks queued now)."""
    if src.is_cuda or src.dtype != torch.float32 or src.dim() != 2:
        raise ValueError("src must be a 2-D float32 host tensor")
    src = src.contiguous()
    n, dim = src.shape
    with torch.cuda.device(dev):
        comp = torch.cuda.current_stream(dev)
        copy = stream if stream is not None else torch.cuda.Stream(dev)
        raw = torch.empty((n, dim), dtype=torch.float32, device=dev)
        copy.wait_stream(comp)   # `raw` was allocated on the compute stream
        return StagedCopy(src, raw, _stream_chunks(n, chunks), copy, src.is_pinned())


def join_streamed(L: PreparedRelation, right_host, theta: float,
                  band: Optional[float] = None, left_base: int = 0, chunks: int = 8,
                  name: str = "", sync: bool = True) -> Tuple["DeviceMatches", PreparedRelation]:
    """join_chunked for a HOST right relation (a tensor, or a StagedCopy whose
    chunk copies are already queued): the rows are copied in chunks on a side
    stream and normalised in place as each chunk lands, so the host->device
    copy overlaps the filter.  Pinned sources copy asynchronously; a pageable
    one blocks the host per chunk while the GPU filters the previous one."""
    staged = right_host if isinstance(right_host, StagedCopy) else stage_host(right_host, L.device,
                                                                           chunks)
    return join_chunked(L, staged.raw, staged.arrive, theta, band, left_base, chunks,
                        inplace=True, name=name, spans=staged.spans, sync=sync)


def prepare_gather(table: torch.Tensor, index: torch.Tensor, name: str = "") -> PreparedRelation:
    """Prepare relation rows table[index[i]] (lookup-model prefetch) in one pass."""
    _check_matrix(table, "table")
    if index.dtype != torch.int64 or not index.is_cuda or index.dim() != 1:
        raise ValueError("index must be a 1-D int64 CUDA tensor")
    L = _lib.lib()
    n, dim = int(index.numel()), table.shape[1]
    dev = table.device
    f32 = torch.empty((n, dim), dtype=torch.float32, device=dev)
    op = op_empty(n, dim, dev)
    rep = torch.zeros(1, dtype=torch.int64, device=dev)
    re, te = _err_buffers(n, dev)
    with torch.cuda.device(dev):
        _lib.check(L.sjb_gather_normalize_rows(_vp(table), _vp(index.contiguous()), n, dim,
                                               _vp(f32), _vp(op), _vp(rep), _vp(re), _vp(te),
                                               _stream(dev)),
                   "sjb_gather_normalize_rows")
    return PreparedRelation(f32, op, n, dim, name, rep, re, te)


def _pack_host(tokens) -> Tuple[np.ndarray, np.ndarray]:
    """UTF-8 bytes (+ NUL) and int64 offsets of the tokens, on the host: the
    native packer (csrc/sjb_pack.c) when built, else an equivalent Python
    path (host-side marshalling only; no computation falls back)."""
    try:
        from . import _sjbpack
    except ImportError:
        _sjbpack = None
    if _sjbpack is not None:
        data, offs = _sjbpack.pack(tokens)
        return np.frombuffer(data, dtype=np.uint8), np.frombuffer(offs, dtype=np.int64)
    n = len(tokens)
    joined = "".join(tokens)
    if joined.isascii():
        raw = joined.encode("ascii")
        lens = np.fromiter(map(len, tokens), dtype=np.int64, count=n)
    else:
        enc = [t.encode("utf-8") for t in tokens]
        raw = b"".join(enc)
        lens = np.fromiter(map(len, enc), dtype=np.int64, count=n)
    offs = np.zeros(n + 1, dtype=np.int64)
    if n:
        np.cumsum(lens, out=offs[1:])
    return np.frombuffer(raw + b"\0", dtype=np.uint8), offs


def pack_tokens(tokens, device: torch.device) -> Tuple[torch.Tensor, torch.Tensor]:
    """UTF-8 bytes of the tokens (device u8) and n+1 int64 offsets (device)."""
    buf, offs = _pack_host(tokens)
    return (torch.from_numpy(buf.copy()).to(device, non_blocking=False),
            torch.from_numpy(offs.copy()).to(device))


def fnv1a64_tokens(tokens, xor_seed: int, device: torch.device) -> torch.Tensor:
    """FNV-1a-64 of every token XOR seed, on the device (int64 holding u64)."""
    b, o = pack_tokens(tokens, device)
    out = torch.empty(len(tokens), dtype=torch.int64, device=device)
    if len(tokens):
        with torch.cuda.device(device):
            _lib.check(_lib.lib().sjb_fnv1a64_many(_vp(b), _vp(o), len(tokens),
                                                   ctypes.c_uint64(xor_seed & (2**64 - 1)),
                                                   _vp(out), _stream(device)),
                       "sjb_fnv1a64_many")
    return out


def synthetic_rows(seeds: torch.Tensor, dim: int) -> torch.Tensor:
    """Synthetic-model rows (normalised) from device u64 stream seeds."""
    dev = seeds.device
    out = torch.empty((seeds.numel(), dim), dtype=torch.float32, device=dev)
    if seeds.numel():
        with torch.cuda.device(dev):
            _lib.check(_lib.lib().sjb_synthetic_fill_many(_vp(seeds), seeds.numel(), dim,
                                                          _vp(out), ctypes.c_void_p(0),
                                                          None, None, _stream(dev)),
                       "sjb_synthetic_fill_many")
    return out


def subword_rows(tokens, table: torch.Tensor, minn: int, maxn: int,
                 prepared: bool = False, name: str = ""):
    """Subword-model rows; prepared=True returns a PreparedRelation (embed +
    normalise + operand image), else the raw (n, dim) embedding."""
    _check_matrix(table, "bucket table")
    dev = table.device
    b, o = pack_tokens(tokens, dev)
    n, dim = len(tokens), table.shape[1]
    f32 = torch.empty((n, dim), dtype=torch.float32, device=dev)
    op = op_empty(n, dim, dev) if prepared else None
    rep = torch.zeros(1, dtype=torch.int64, device=dev)
    re, te = _err_buffers(n, dev) if prepared else (None, None)
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().sjb_subword_embed(_vp(b), _vp(o), n, _vp(table), table.shape[0],
                                                dim, minn, maxn, 1 if prepared else 0,
                                                _vp(f32), _vp(op), _vp(rep), _vp(re), _vp(te),
                                                _stream(dev)),
                   "sjb_subword_embed")
    if prepared:
        return PreparedRelation(f32, op, n, dim, name, rep, re, te)
    return f32
