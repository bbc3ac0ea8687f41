"""The reference's own CPU join path, driven from its compiled C kernels.

TEST / BASELINE INFRASTRUCTURE ONLY (bench.py ``--impl reference`` and the
``cpu_baseline`` leg, plus tests that cross-check the oracle).  The product
package never imports this module.

``oracle/_ref/libref_v{4,3}.so`` is the reference's ``_kernelcore.c`` compiled
in place from /root/reference by ``oracle/Makefile`` (outputs only into
``oracle/_ref/``, git-ignored, shipped to the GPU box with the snapshot).  The
reference's orchestration above those kernels is thin Python; it cannot
travel to the GPU box (no /root/reference there), so it is restated here
line for line:

* ``plan_batches``   <- join.py:88-108
* ``_exec_tiles``    <- join.py:297-314 (``_EXEC_CHUNK_ELEMS`` = 2**19, join.py:48)
* ``tensor_join_vectors`` <- join.py:317-373 with the prefetched vectors already
  embedded (LookupModel path): normalize_rows (linalg.py:87-98) ->
  pack_transpose (join.py:342) -> per-worker tile_dot + scan_hits
  (linalg.py:116-153, _ckern.pyx:131-176) over round-robin tiles on Python
  threads (join.py:121-142, 339-359) -> MatchSink.merge/canonicalize
  (core.py:178-213).
* ``nlj_rows``       <- _ckern.pyx:179-212 (hit-buffer resume protocol).

ctypes releases the GIL for the duration of each foreign call, exactly like
the Cython wrappers' ``with nogil`` blocks, so worker threads run the C
kernels in parallel as they do in the reference.
"""

from __future__ import annotations

import ctypes
import math
import os
import threading
import time
from typing import List, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_REF_DIR = os.path.join(_HERE, "_ref")

_c_f32p = ctypes.POINTER(ctypes.c_float)
_c_u64p = ctypes.POINTER(ctypes.c_uint64)
_c_long = ctypes.c_long

EXEC_CHUNK_ELEMS = 1 << 19          # join.py:48
PREFILTER_BAND = 1e-4               # join.py:44
DEFAULT_BUDGET = 64 * 1024 * 1024   # cli.py:31


def _cpu_has_avx512() -> bool:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("flags"):
                    return " avx512f " in (line + " ")
    except OSError:
        pass
    return False


_lib = None
_variant = None


def available() -> bool:
    return any(os.path.exists(os.path.join(_REF_DIR, f))
               for f in ("libref_v4.so", "libref_v3.so"))


def variant() -> str:
    lib()
    return _variant


def lib():
    """Load the reference kernel library built for this host's ISA."""
    global _lib, _variant
    if _lib is not None:
        return _lib
    order = ["libref_v4.so", "libref_v3.so"] if _cpu_has_avx512() else ["libref_v3.so"]
    path = None
    for name in order:
        cand = os.path.join(_REF_DIR, name)
        if os.path.exists(cand):
            path = cand
            break
    if path is None:
        raise FileNotFoundError(
            f"reference kernels not built under {_REF_DIR}; run `make -C oracle ref` "
            "in a container that has /root/reference")
    L = ctypes.CDLL(path)
    L.sj_normalize_rows.restype = _c_long
    L.sj_normalize_rows.argtypes = [_c_f32p, _c_long, _c_long]
    L.sj_pack_transpose.argtypes = [_c_f32p, _c_long, _c_long, _c_f32p]
    L.sj_tile_dot.argtypes = [_c_f32p, _c_long, _c_f32p, _c_long, _c_long, _c_long,
                              _c_long, _c_f32p, _c_long]
    L.sj_scan_count.restype = _c_long
    L.sj_scan_count.argtypes = [_c_f32p, _c_long, ctypes.c_float]
    L.sj_scan_fill.restype = _c_long
    L.sj_scan_fill.argtypes = [_c_f32p, _c_long, _c_long, ctypes.c_float,
                               ctypes.c_uint64, ctypes.c_uint64, _c_u64p, _c_u64p,
                               _c_f32p]
    L.sj_dot_seq.restype = ctypes.c_float
    L.sj_dot_seq.argtypes = [_c_f32p, _c_f32p, _c_long]
    L.sj_nlj_rows.restype = _c_long
    L.sj_nlj_rows.argtypes = [_c_f32p, _c_long, _c_long, _c_f32p, _c_long, _c_long,
                              ctypes.c_float, ctypes.c_float, _c_u64p, _c_u64p,
                              _c_f32p, _c_long, ctypes.POINTER(_c_long)]
    L.sj_fnv1a64.restype = ctypes.c_uint64
    L.sj_fnv1a64.argtypes = [ctypes.POINTER(ctypes.c_ubyte), _c_long]
    L.sj_synthetic_fill.argtypes = [ctypes.c_uint64, _c_long, _c_f32p]
    _lib = L
    _variant = os.path.basename(path)
    return L


def _p(a, t):
    return a.ctypes.data_as(t)


def normalize_rows(m: np.ndarray) -> Tuple[np.ndarray, int]:
    out = np.ascontiguousarray(m, dtype=np.float32).copy()
    if out.size == 0:
        return out, 0
    return out, int(lib().sj_normalize_rows(_p(out, _c_f32p), out.shape[0],
                                            out.shape[1]))


def fnv1a64(data: bytes) -> int:
    buf = (ctypes.c_ubyte * max(1, len(data))).from_buffer_copy(bytes(data) + b"\0")
    return int(lib().sj_fnv1a64(buf, len(data)))


def synthetic_fill(seed: int, dim: int) -> np.ndarray:
    out = np.empty(dim, dtype=np.float32)
    lib().sj_synthetic_fill(ctypes.c_uint64(seed & (2**64 - 1)), dim, _p(out, _c_f32p))
    return out


def dot_seq(a, b) -> np.float32:
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    return np.float32(lib().sj_dot_seq(_p(a, _c_f32p), _p(b, _c_f32p), a.shape[0]))


def plan_batches(left_rows: int, right_rows: int, budget_bytes: int):
    """join.py:88-108 -> list of (ls, lc, rs, rc)."""
    if budget_bytes < 4:
        raise ValueError(f"budget {budget_bytes} bytes cannot hold one fp32 cell")
    budget_elems = budget_bytes // 4
    b = math.isqrt(budget_elems)
    left_block = max(1, min(b, left_rows))
    right_block = max(1, min(budget_elems // left_block, right_rows))
    tiles = []
    for ls in range(0, left_rows, left_block):
        lc = min(left_block, left_rows - ls)
        for rs in range(0, right_rows, right_block):
            tiles.append((ls, lc, rs, min(right_block, right_rows - rs)))
    return tiles


def exec_tiles(tiles):
    """join.py:297-314."""
    out = []
    for (ls, lc, rs, rc) in tiles:
        rows_cap = max(1, EXEC_CHUNK_ELEMS // rc)
        if rows_cap > 12:
            rows_cap -= rows_cap % 12
        if rows_cap >= lc:
            out.append((ls, lc, rs, rc))
            continue
        for s in range(ls, ls + lc, rows_cap):
            out.append((s, min(rows_cap, ls + lc - s), rs, rc))
    return out


def canonicalize(lefts, rights, sims):
    """core.py:196-213."""
    if len(lefts) == 0:
        return lefts, rights, sims
    order = np.lexsort((rights, lefts))
    lefts, rights, sims = lefts[order], rights[order], sims[order]
    keep = np.ones(len(lefts), dtype=bool)
    keep[1:] = (lefts[1:] != lefts[:-1]) | (rights[1:] != rights[:-1])
    return (np.ascontiguousarray(lefts[keep]), np.ascontiguousarray(rights[keep]),
            np.ascontiguousarray(sims[keep]))


def _run_workers(n, target):
    """join.py:121-142."""
    if n <= 1:
        target(0)
        return
    failures: List[BaseException] = []

    def run(w):
        try:
            target(w)
        except BaseException as exc:  # noqa: BLE001
            failures.append(exc)

    ts = [threading.Thread(target=run, args=(w,)) for w in range(n)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if failures:
        raise failures[0]


def pack_transpose(nr: np.ndarray) -> np.ndarray:
    """sj_pack_transpose (_kernelcore.c:113-117), done once per join (join.py:342)."""
    packed = np.empty((nr.shape[1], nr.shape[0]), dtype=np.float32)
    lib().sj_pack_transpose(_p(nr, _c_f32p), nr.shape[0], nr.shape[1], _p(packed, _c_f32p))
    return packed


def tensor_join_normalized(nl: np.ndarray, nr: np.ndarray, theta: float,
                           budget_bytes: int = DEFAULT_BUDGET, threads: int = 1,
                           left_offset: int = 0, packed: np.ndarray = None,
                           plan_rows: int = None):
    """tensor_join (join.py:317-373) after embed+normalize: tiles, workers, merge.

    ``left_offset`` shifts emitted left offsets (used for bounded row samples
    of a larger relation); ``packed`` passes a pack_transpose of ``nr`` made
    once for several row samples.  ``plan_rows`` plans the tile grid for a
    relation of that many left rows and executes only the tiles that fall in
    the rows given (a bounded sample runs exactly the full job's first tiles).
    Returns (lefts, rights, sims, peak_buffer_bytes).
    """
    L = lib()
    theta32 = ctypes.c_float(np.float32(theta))
    dim = nl.shape[1]
    n_plan = nl.shape[0] if plan_rows is None else max(plan_rows, nl.shape[0])
    tiles = exec_tiles(plan_batches(n_plan, nr.shape[0], budget_bytes))
    if n_plan != nl.shape[0]:
        tiles = [(ls, min(lc, nl.shape[0] - ls), rs, rc) for (ls, lc, rs, rc) in tiles
                 if ls < nl.shape[0]]
    n_workers = max(1, min(threads, len(tiles)))
    assignments = [tiles[w::n_workers] for w in range(n_workers)]
    parts: List[list] = [[] for _ in range(n_workers)]
    buffer_bytes = [0] * n_workers
    if tiles and packed is None:
        packed = pack_transpose(nr)
    ldb = nr.shape[0]

    def work(w):
        mine = assignments[w]
        if not mine:
            return
        cap = max(lc * rc for (_, lc, _, rc) in mine)
        buf = np.empty(cap, dtype=np.float32)
        buffer_bytes[w] = buf.nbytes
        bp = buf.ctypes.data
        for (ls, lc, rs, rc) in mine:
            left_ptr = ctypes.cast(nl.ctypes.data + ls * dim * 4, _c_f32p)
            bt_ptr = ctypes.cast(packed.ctypes.data + rs * 4, _c_f32p)
            L.sj_tile_dot(left_ptr, dim, bt_ptr, ldb, lc, rc, dim,
                          ctypes.cast(bp, _c_f32p), rc)
            k = L.sj_scan_count(ctypes.cast(bp, _c_f32p), lc * rc, theta32)
            if k == 0:
                continue
            lo = np.empty(k, dtype=np.uint64)
            ro = np.empty(k, dtype=np.uint64)
            so = np.empty(k, dtype=np.float32)
            L.sj_scan_fill(ctypes.cast(bp, _c_f32p), lc, rc, theta32,
                           ctypes.c_uint64(ls + left_offset), ctypes.c_uint64(rs),
                           _p(lo, _c_u64p), _p(ro, _c_u64p), _p(so, _c_f32p))
            parts[w].append((lo, ro, so))

    if tiles:
        _run_workers(n_workers, work)
    flat = [c for p in parts for c in p]
    if not flat:
        e = np.empty(0, dtype=np.uint64)
        return e, e.copy(), np.empty(0, dtype=np.float32), sum(buffer_bytes)
    lefts = np.concatenate([c[0] for c in flat])
    rights = np.concatenate([c[1] for c in flat])
    sims = np.concatenate([c[2] for c in flat])
    lo, ro, so = canonicalize(lefts, rights, sims)
    return lo, ro, so, sum(buffer_bytes)


def tensor_join_vectors(L_raw: np.ndarray, S_raw: np.ndarray, theta: float,
                        budget_bytes: int = DEFAULT_BUDGET, threads: int = 1):
    """Full reference tensor join over prefetched vectors; returns
    (lefts, rights, sims, stats) with stats wall/normalize/join nanos."""
    t0 = time.perf_counter_ns()
    nl, _ = normalize_rows(L_raw)
    nr, _ = normalize_rows(S_raw)
    t1 = time.perf_counter_ns()
    lo, ro, so, peak = tensor_join_normalized(nl, nr, theta, budget_bytes, threads)
    t2 = time.perf_counter_ns()
    return lo, ro, so, {"wall_nanos": t2 - t0, "normalize_nanos": t1 - t0,
                        "join_nanos": t2 - t1, "peak_buffer_bytes": peak,
                        "threads": threads, "variant": _variant}


def nlj_rows(left: np.ndarray, i0: int, i1: int, right: np.ndarray, theta: float,
             band: float = PREFILTER_BAND):
    """_ckern.pyx:179-212: row-at-a-time join with the hit-buffer resume loop."""
    L = lib()
    ns, dim = right.shape
    chunks = []
    if ns == 0 or i0 >= i1:
        return chunks
    cap = max(4 * ns, 32768)
    oi = np.empty(cap, dtype=np.uint64)
    oj = np.empty(cap, dtype=np.uint64)
    os_ = np.empty(cap, dtype=np.float32)
    nxt = _c_long(0)
    row = i0
    while row < i1:
        k = L.sj_nlj_rows(_p(left, _c_f32p), row, i1, _p(right, _c_f32p), ns, dim,
                          ctypes.c_float(np.float32(theta)),
                          ctypes.c_float(np.float32(band)),
                          _p(oi, _c_u64p), _p(oj, _c_u64p), _p(os_, _c_f32p), cap,
                          ctypes.byref(nxt))
        if k > 0:
            chunks.append((oi[:k].copy(), oj[:k].copy(), os_[:k].copy()))
        if nxt.value == row:
            raise MemoryError("hit buffer smaller than one row")
        row = nxt.value
    return chunks
