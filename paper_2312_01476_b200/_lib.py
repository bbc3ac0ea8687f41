"""ctypes binding of libsjb200.so (the C ABI in include/simjoin_b200.h).

The product path has no fallback: if the library is missing or fails to load,
:func:`lib` raises, and every operator that needs the GPU raises with it.
"""

from __future__ import annotations

import ctypes
import os

from .build import LIB_PATH

EXPORTS = (
    "sjb_version", "sjb_last_error", "sjb_launch_count", "sjb_sm_count", "sjb_kpad", "sjb_operand_elems",
    "sjb_normalize_rows", "sjb_gather_normalize_rows", "sjb_cast_rows", "sjb_prepare_bf16", "sjb_raw_band", "sjb_ab_kernels", "sjb_debug_blk_stats", "sjb_row_norms", "sjb_fnv1a64_many", "sjb_synthetic_fill_many",
    "sjb_subword_embed", "sjb_join_workspace_bytes", "sjb_default_band", "sjb_accum_slack",
    "sjb_tile_count", "sjb_join_begin", "sjb_join_filter_tiles", "sjb_join_finish",
    "sjb_join_prepared_async", "sjb_join_prepared", "sjb_tile_dot", "sjb_dots_vm", "sjb_cosine_vm",
    "sjb_scan_hits", "sjb_scan_hits_workspace_bytes",
    "sjb_matches_csv_workspace_bytes", "sjb_matches_csv_layout", "sjb_matches_csv_write",
)

SJB_OK = 0


class JoinArgs(ctypes.Structure):
    _fields_ = [
        ("n_left", ctypes.c_int64), ("n_right", ctypes.c_int64), ("dim", ctypes.c_int64),
        ("theta", ctypes.c_float), ("band", ctypes.c_float),
        ("cand_cap", ctypes.c_int64), ("out_cap", ctypes.c_int64),
        ("left_base", ctypes.c_uint64),
        ("grid", ctypes.c_int32), ("tiles_per_chunk", ctypes.c_int32),
        ("ev_filter_begin", ctypes.c_void_p), ("ev_filter_end", ctypes.c_void_p),
        ("left_row_err", ctypes.c_void_p), ("right_tile_err", ctypes.c_void_p),
        ("recheck", ctypes.c_int32),
        ("left_inv_norm", ctypes.c_void_p), ("right_inv_norm", ctypes.c_void_p),
        ("sims_mode", ctypes.c_int32), ("launch_grid", ctypes.c_int32),
    ]


class JoinInfo(ctypes.Structure):
    _fields_ = [
        ("n_matches", ctypes.c_int64), ("n_candidates", ctypes.c_int64),
        ("cand_needed", ctypes.c_int64), ("overflow", ctypes.c_int32), ("grid", ctypes.c_int32),
    ]


class SjbError(RuntimeError):
    """A C-ABI call returned a non-zero status."""


_lib = None

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64


def lib(path: str = LIB_PATH):
    """Load (once) and return the library handle with typed signatures."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is not built; run `python -m paper_2312_01476_b200.build` "
            "(or __graft_entry__.build()) first -- there is no CPU fallback")
    L = ctypes.CDLL(path)
    L.sjb_version.restype = ctypes.c_int
    L.sjb_launch_count.restype = ctypes.c_int64
    L.sjb_last_error.restype = ctypes.c_char_p
    L.sjb_sm_count.restype = ctypes.c_int
    L.sjb_sm_count.argtypes = [ctypes.c_int]
    L.sjb_kpad.restype = _i64
    L.sjb_kpad.argtypes = [_i64]
    L.sjb_operand_elems.restype = _i64
    L.sjb_operand_elems.argtypes = [_i64, _i64]
    L.sjb_default_band.restype = ctypes.c_float
    L.sjb_default_band.argtypes = [_i64]
    L.sjb_accum_slack.restype = ctypes.c_float
    L.sjb_accum_slack.argtypes = [_i64]
    L.sjb_tile_count.restype = _i64
    L.sjb_tile_count.argtypes = [_i64]
    L.sjb_normalize_rows.argtypes = [_vp, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp]
    L.sjb_gather_normalize_rows.argtypes = [_vp, _vp, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp]
    L.sjb_row_norms.argtypes = [_vp, _i64, _i64, _vp, _vp]
    L.sjb_cast_rows.argtypes = [_vp, _i64, _i64, _vp, _vp]
    L.sjb_prepare_bf16.argtypes = [_vp, _i64, _i64, _vp, _vp, _vp, _vp, _vp]
    L.sjb_raw_band.argtypes = [_i64]
    L.sjb_raw_band.restype = ctypes.c_float
    L.sjb_ab_kernels.restype = ctypes.c_int
    L.sjb_debug_blk_stats.argtypes = [_vp]
    L.sjb_fnv1a64_many.argtypes = [_vp, _vp, _i64, ctypes.c_uint64, _vp, _vp]
    L.sjb_synthetic_fill_many.argtypes = [_vp, _i64, _i64, _vp, _vp, _vp, _vp, _vp]
    L.sjb_subword_embed.argtypes = [_vp, _vp, _i64, _vp, _i64, _i64, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_int, _vp, _vp, _vp, _vp, _vp, _vp]
    L.sjb_join_workspace_bytes.restype = _i64
    L.sjb_join_workspace_bytes.argtypes = [ctypes.POINTER(JoinArgs)]
    L.sjb_join_prepared_async.argtypes = [_vp, _vp, _vp, _vp, ctypes.POINTER(JoinArgs), _vp, _i64,
                                          _vp, _vp, _vp, _vp, _vp]
    L.sjb_join_begin.argtypes = [ctypes.POINTER(JoinArgs), _vp, _i64, _vp]
    L.sjb_join_filter_tiles.argtypes = [_vp, _vp, _vp, _vp, ctypes.POINTER(JoinArgs), _vp, _i64,
                                        _i64, _i64, _vp]
    L.sjb_join_finish.argtypes = [_vp, _vp, ctypes.POINTER(JoinArgs), _vp, _i64, _vp, _vp, _vp,
                                  _vp, _vp]
    L.sjb_join_prepared.argtypes = [_vp, _vp, _vp, _vp, ctypes.POINTER(JoinArgs), _vp, _i64,
                                    _vp, _vp, _vp, ctypes.POINTER(JoinInfo), _vp]
    L.sjb_tile_dot.argtypes = [_vp, _i64, _vp, _i64, _i64, _i64, _i64, _vp, _i64, _vp]
    L.sjb_dots_vm.argtypes = [_vp, _vp, _i64, _i64, _vp, _vp]
    L.sjb_cosine_vm.argtypes = [_vp, _vp, _i64, _i64, _vp, _vp, _vp]
    L.sjb_scan_hits.argtypes = [_vp, _i64, _i64, ctypes.c_float, ctypes.c_uint64,
                                ctypes.c_uint64, _vp, _vp, _vp, _i64, ctypes.POINTER(_i64),
                                _vp, _i64, _vp]
    L.sjb_scan_hits_workspace_bytes.restype = _i64
    L.sjb_scan_hits_workspace_bytes.argtypes = [_i64]
    L.sjb_matches_csv_workspace_bytes.restype = _i64
    L.sjb_matches_csv_workspace_bytes.argtypes = [_i64]
    L.sjb_matches_csv_layout.argtypes = [_vp, _vp, _vp, _i64, _vp, _i64, ctypes.POINTER(_i64), _vp]
    L.sjb_matches_csv_write.argtypes = [_vp, _vp, _vp, _i64, _vp, _i64, _vp, _i64, _vp]
    for name in EXPORTS:
        if not hasattr(L, name):
            raise ImportError(f"{path} does not export {name}")
    _lib = L
    return L


def check(rc: int, what: str) -> None:
    if rc != SJB_OK:
        msg = lib().sjb_last_error()
        raise SjbError(f"{what}: status {rc}: {msg.decode() if msg else ''}")
