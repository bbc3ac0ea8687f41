"""Vector-against-relation cosine on the device (reference linalg.py:55-84).

``cosine_vm`` keeps the reference's arithmetic bit for bit: the sequential
fmaf dot (sj_dots_vm), norms as fp64 sequential sums rounded to fp32
(sj_row_norms), then fp32 ``na * norm_i`` and fp32 ``dot / denom``, all in one
kernel (``sjb_cosine_vm``).  It is the primitive of ``e_selection``
(join.py) and ``top_k`` (embedding.py).  No CPU fallback.
"""

from __future__ import annotations

import ctypes
from typing import Optional, Union

import numpy as np
import torch

from . import _lib
from . import device as D
from .core import EmbeddedRelation, check_dims
from .errors import ZeroVector


def _as_f32_vector(a) -> np.ndarray:
    arr = np.ascontiguousarray(a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else a,
                               dtype=np.float32)
    if arr.ndim != 1:
        raise ValueError(f"expected a vector, got shape {arr.shape}")
    return arr


def cosine_vm_device(a, m: torch.Tensor) -> torch.Tensor:
    """Cosine of vector `a` against every row of the (n, dim) CUDA tensor `m`
    (a device fp32 tensor of n sims).  Raises ZeroVector like the reference
    (zero-norm probe, or a zero-norm row)."""
    if not m.is_cuda or m.dtype != torch.float32 or m.dim() != 2:
        raise ValueError("m must be a 2-D float32 CUDA tensor")
    n, dim = m.shape
    dev = m.device
    if isinstance(a, torch.Tensor) and a.is_cuda:   # stays on the device
        if a.dim() != 1:
            raise ValueError(f"expected a vector, got shape {tuple(a.shape)}")
        check_dims(a.shape[0], dim)
        ta = a.to(device=dev, dtype=torch.float32).contiguous()
    else:
        va = _as_f32_vector(a)
        check_dims(va.shape[0], dim)
        ta = torch.from_numpy(va).to(dev)
    m = m.contiguous()
    out = torch.empty(n, dtype=torch.float32, device=dev)
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    if dim == 0:
        raise ZeroVector("cosine of a zero-norm vector")
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().sjb_cosine_vm(D._vp(ta), D._vp(m), n, dim, D._vp(out),
                                            D._vp(flags), D._stream(dev)), "sjb_cosine_vm")
    f = int(flags.item())
    if f & 1:
        raise ZeroVector("cosine of a zero-norm vector")
    if f & 2:
        raise ZeroVector("relation contains a zero-norm row")
    return out


def cosine_vm(a, m: Union[EmbeddedRelation, np.ndarray, torch.Tensor],
              device=None) -> np.ndarray:
    """Element i = cosine_vv(a, row i) (reference linalg.py:70-84)."""
    if isinstance(m, EmbeddedRelation):
        data = m.data
    else:
        data = m
    if isinstance(data, torch.Tensor) and data.is_cuda:
        t = data
    else:
        dev = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        arr = np.ascontiguousarray(data, dtype=np.float32)
        if not arr.flags.writeable:          # EmbeddedRelation data is read-only
            arr = arr.copy()
        t = torch.from_numpy(arr).to(dev)
    return cosine_vm_device(a, t).cpu().numpy()
