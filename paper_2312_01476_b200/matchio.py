"""The matches file, formatted on the GPU.

The reference writes a join's result as text, one line per match
(cli._write_matches, cli.py:105-108):

    f"{left},{right},{_fmt_sim(sim)}\\n"

with ``_fmt_sim`` = ``numpy.format_float_positional(float32(sim),
unique=True, trim="-")`` (cli.py:99-102), the shortest positional decimal
that reads back as the same float32.  Its Python loop costs ~microseconds
per line.  Here the bytes are produced by two kernels of libsjb200.so
(csrc/sjb_fmt.cu: line lengths per 256-line group -> scan -> text), from
match columns already on the device, so a join's MatchSet goes to a file
without a per-line host loop.  The result is byte-identical to the
reference writer (tests/test_gpu_parity.py::test_matches_file_*).
"""
from __future__ import annotations

import ctypes
import warnings
from typing import Union

import numpy as np
import torch

from . import _lib
from . import device as D
from .core import MatchSet


def format_columns_device(lefts: torch.Tensor, rights: torch.Tensor,
                          sims: torch.Tensor) -> torch.Tensor:
    """The matches file of device columns (int64 tensors holding u64 offsets,
    float32 sims) as a uint8 CUDA tensor, on the current stream."""
    for t, dt, what in ((lefts, torch.int64, "lefts"), (rights, torch.int64, "rights"),
                        (sims, torch.float32, "sims")):
        if not t.is_cuda or t.dtype != dt or t.dim() != 1:
            raise ValueError(f"{what} must be a 1-D {dt} CUDA tensor")
    n = lefts.numel()
    if rights.numel() != n or sims.numel() != n:
        raise ValueError("match columns must have equal length")
    dev = lefts.device
    if n == 0:
        return torch.empty(0, dtype=torch.uint8, device=dev)
    L = _lib.lib()
    lefts, rights, sims = lefts.contiguous(), rights.contiguous(), sims.contiguous()
    with torch.cuda.device(dev):
        wsb = int(L.sjb_matches_csv_workspace_bytes(n))
        ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
        total = ctypes.c_int64(0)
        st = D._stream(dev)
        _lib.check(L.sjb_matches_csv_layout(D._vp(lefts), D._vp(rights), D._vp(sims), n,
                                            D._vp(ws), wsb, ctypes.byref(total), st),
                   "sjb_matches_csv_layout")
        out = torch.empty(total.value, dtype=torch.uint8, device=dev)
        _lib.check(L.sjb_matches_csv_write(D._vp(lefts), D._vp(rights), D._vp(sims), n,
                                           D._vp(ws), wsb, D._vp(out), total.value, st),
                   "sjb_matches_csv_write")
    return out


def _columns(matches, device) -> tuple:
    if isinstance(matches, D.DeviceMatches):
        return matches.lefts, matches.rights, matches.sims
    if isinstance(matches, MatchSet):
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None \
            else torch.device(device)
        cols = []
        for a, npt in ((matches.lefts, np.int64), (matches.rights, np.int64),
                       (matches.sims, np.float32)):
            with warnings.catch_warnings():   # MatchSet columns are read-only; only read here
                warnings.simplefilter("ignore", UserWarning)
                h = torch.from_numpy(np.ascontiguousarray(a).view(npt))
            cols.append(h.to(dev, non_blocking=False))
        return tuple(cols)
    raise TypeError("matches must be a MatchSet or DeviceMatches")


def _format_host(matches, device) -> np.ndarray:
    D.require_cuda()
    out = format_columns_device(*_columns(matches, device))
    if out.numel() == 0:
        return np.empty(0, dtype=np.uint8)
    h = torch.empty(out.numel(), dtype=torch.uint8, pin_memory=True)
    h.copy_(out, non_blocking=True)
    torch.cuda.current_stream(out.device).synchronize()
    return h.numpy()


def format_matches(matches: Union[MatchSet, "D.DeviceMatches"], device=None) -> bytes:
    """The reference's matches-file bytes for a MatchSet (host columns are
    copied to the GPU) or DeviceMatches (formatted in place)."""
    return _format_host(matches, device).tobytes()


def write_matches(path: str, matches: Union[MatchSet, "D.DeviceMatches"], device=None) -> None:
    """cli._write_matches (cli.py:105-108): write the matches file at `path`."""
    data = _format_host(matches, device)
    with open(path, "wb") as fh:
        fh.write(memoryview(data))
