"""``cuda`` kernel backend for the reference's backend registry.

The reference selects kernels through ``simjoin.kernels`` (kernels.py:18-60):
a backend is a module with ``NAME`` and the function set of _ckern.pyx:41-212.
This module provides that set on host numpy arrays, executing every function
with the libsjb200.so kernels (host->device copy, kernel, device->host
copy).  Register it into a reference installation with::

    from paper_2312_01476_b200 import kernels as cuda_backend
    cuda_backend.register(simjoin.kernels)          # adds _BACKENDS["cuda"]
    simjoin.kernels.set_backend("cuda")

after which the reference's own ``backend`` test fixture and ``backends``
benchmark pick it up.  Results are bitwise those of the compiled (FMA)
reference backend: the canonical similarity is the sequential fmaf chain.
"""

from __future__ import annotations

import ctypes
from typing import List, Tuple

import numpy as np
import torch

from . import _lib
from . import device as D
from .embedding import fnv1a64 as _fnv_host

NAME = "cuda"


def _dev() -> torch.device:
    D.require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def _h2d(a: np.ndarray) -> torch.Tensor:
    a = np.ascontiguousarray(a)
    if not a.flags.writeable:          # read-only views (EmbeddedRelation data): copy
        a = a.copy()
    return torch.from_numpy(a).to(_dev())


def _stream():
    return D._stream(_dev())


def fnv1a64(data: bytes) -> int:
    """Single-token hash (scalar; the batch path is device-side)."""
    return _fnv_host(bytes(data))


def synthetic_fill(stream_seed, out: np.ndarray) -> None:
    if out.shape[0] == 0:
        return
    seeds = torch.tensor([np.uint64(int(stream_seed) & (2**64 - 1)).view(np.int64)],
                         dtype=torch.int64, device=_dev())
    out[:] = D.synthetic_rows(seeds, out.shape[0]).cpu().numpy()[0]


def synthetic_fill_many(seeds: np.ndarray, out: np.ndarray) -> None:
    n, dim = out.shape
    if n == 0 or dim == 0:
        return
    s = _h2d(np.ascontiguousarray(seeds, dtype=np.uint64).view(np.int64))
    out[:, :] = D.synthetic_rows(s, dim).cpu().numpy()


def normalize_rows_inplace(m: np.ndarray) -> int:
    n, dim = m.shape
    if n == 0 or dim == 0:
        return 0
    t = _h2d(m.astype(np.float32, copy=False))
    rep = D.normalize_rows_(t)
    m[:, :] = t.cpu().numpy()
    return int(rep.item())


def row_norms(m: np.ndarray) -> np.ndarray:
    n, dim = m.shape
    if n == 0:
        return np.empty(0, dtype=np.float32)
    if dim == 0:
        return np.zeros(n, dtype=np.float32)
    t = _h2d(m.astype(np.float32, copy=False))
    out = torch.empty(n, dtype=torch.float32, device=t.device)
    _lib.check(_lib.lib().sjb_row_norms(D._vp(t), n, dim, D._vp(out), _stream()),
               "sjb_row_norms")
    return out.cpu().numpy()


def dots_vm(a: np.ndarray, m: np.ndarray) -> np.ndarray:
    n, dim = m.shape
    if n == 0:
        return np.empty(0, dtype=np.float32)
    if dim == 0:
        return np.zeros(n, dtype=np.float32)
    ta, tm = _h2d(a.astype(np.float32, copy=False)), _h2d(m.astype(np.float32, copy=False))
    out = torch.empty(n, dtype=torch.float32, device=tm.device)
    _lib.check(_lib.lib().sjb_dots_vm(D._vp(ta), D._vp(tm), n, dim, D._vp(out), _stream()),
               "sjb_dots_vm")
    return out.cpu().numpy()


def dot_seq(a: np.ndarray, b: np.ndarray) -> float:
    if a.shape[0] == 0:
        return 0.0
    return float(dots_vm(a, b.reshape(1, -1))[0])


def pack_transpose(m: np.ndarray) -> np.ndarray:
    """d x n transpose of the right relation (pure layout; device copy)."""
    n, dim = m.shape
    if n == 0 or dim == 0:
        return np.empty((dim, n), dtype=np.float32)
    return _h2d(m).t().contiguous().cpu().numpy()


def tile_dot(left: np.ndarray, bt: np.ndarray, out: np.ndarray) -> None:
    """out[i, j] = canonical dot(left[i], bt[:, j]) (sj_tile_dot)."""
    nl, dim = left.shape
    nr = bt.shape[1]
    if nl == 0 or nr == 0:
        return
    if bt.strides[1] != 4:
        raise ValueError("packed right matrix must be row-contiguous")
    tl = _h2d(left)
    tb = _h2d(bt)                       # contiguous copy: ldb = nr
    to = torch.empty((nl, nr), dtype=torch.float32, device=tl.device)
    _lib.check(_lib.lib().sjb_tile_dot(D._vp(tl), dim, D._vp(tb), nr, nl, nr, dim, D._vp(to), nr,
                                       _stream()), "sjb_tile_dot")
    out[:, :] = to.cpu().numpy()


def scan_hits(buf: np.ndarray, theta, left0, right0
              ) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
    """(left, right, sim) of every cell >= theta in row-major order."""
    nl, nr = buf.shape
    empty = (np.empty(0, dtype=np.uint64), np.empty(0, dtype=np.uint64),
             np.empty(0, dtype=np.float32))
    if nl == 0 or nr == 0:
        return empty
    L = _lib.lib()
    tb = _h2d(buf.astype(np.float32, copy=False))
    wsb = int(L.sjb_scan_hits_workspace_bytes(nl))
    ws = torch.empty(wsb, dtype=torch.uint8, device=tb.device)
    count = ctypes.c_int64(0)
    th = ctypes.c_float(np.float32(theta))
    l0, r0 = ctypes.c_uint64(int(left0)), ctypes.c_uint64(int(right0))
    null = ctypes.c_void_p(0)
    _lib.check(L.sjb_scan_hits(D._vp(tb), nl, nr, th, l0, r0, null, null, null, 0,
                               ctypes.byref(count), D._vp(ws), wsb, _stream()), "sjb_scan_hits")
    k = count.value
    if k == 0:
        return empty
    lo = torch.empty(k, dtype=torch.int64, device=tb.device)
    ro = torch.empty_like(lo)
    so = torch.empty(k, dtype=torch.float32, device=tb.device)
    _lib.check(L.sjb_scan_hits(D._vp(tb), nl, nr, th, l0, r0, D._vp(lo), D._vp(ro), D._vp(so), k,
                               ctypes.byref(count), D._vp(ws), wsb, _stream()), "sjb_scan_hits")
    return (lo.cpu().numpy().view(np.uint64), ro.cpu().numpy().view(np.uint64),
            so.cpu().numpy())


def nlj_rows(left: np.ndarray, i0: int, i1: int, right: np.ndarray, theta: float,
             band: float) -> List[Tuple[np.ndarray, np.ndarray, np.ndarray]]:
    """Row-at-a-time join contract (_ckern.pyx:179-212) of normalised rows
    [i0, i1) against `right`, as one canonical chunk.  `band` is the CPU
    prefilter slack of the reference; the device filter uses its own
    provable band and rechecks canonically, so decisions are identical."""
    ns = right.shape[0]
    if ns == 0 or i0 >= i1:
        return []
    tl = _h2d(np.ascontiguousarray(left[i0:i1], dtype=np.float32))
    tr = _h2d(np.ascontiguousarray(right, dtype=np.float32))
    # the rows are used as given (the contract passes normalised rows, but
    # any rows are accepted): the operand image is their own cast and the
    # band covers their norms, so the canonical recheck sees every pair
    # whose raw dot can reach theta
    pl, pr = D.cast_prepared(tl), D.cast_prepared(tr)
    b = D.band_for_rows(left.shape[1], D.max_row_norm(tl), D.max_row_norm(tr))
    if not np.isfinite(b):
        b = 4.0 * max(1.0, abs(float(theta))) + 1e30      # cutoff below every finite dot
    m = D.join_prepared(pl, pr, float(theta), band=b, left_base=i0)
    if m.n_matches == 0:
        return []
    return [m.to_host()]


def register(kernels_module) -> None:
    """Install this backend into a reference ``simjoin.kernels`` module."""
    kernels_module._BACKENDS[NAME] = __import__(__name__, fromlist=["NAME"])
