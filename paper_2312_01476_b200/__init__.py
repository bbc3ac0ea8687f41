"""simjoin-b200: B200-native cosine-threshold tensor join.

The hot path of arXiv 2312.01476's context-enhanced join (prefetch ->
normalise-and-cast -> fused tcgen05 filter -> canonical fp32 recheck ->
compaction -> R-sharded multi-GPU), exposed through the reference
``simjoin`` package's join/embedding API so it drops in for it.  Names below
mirror the reference's ``__all__`` (reference __init__.py:67-110) for the
components on the hot path.

Importing the package needs no GPU; calling a join does (there is no CPU
fallback).
"""

from .core import (EmbeddedRelation, MatchSet, MatchSink, RawRelation, Threshold, canonicalize,
                   make_raw_relation)
from .errors import (BudgetTooSmall, BufferTooSmall, CapacityExceeded, DimensionMismatch,
                     OffsetOutOfRange, OutOfVocabulary, ParseError, SimjoinError, ZeroVector)

__version__ = "0.1.0"

_LAZY = {
    # join operators (need torch + the CUDA library)
    "BatchPlan": "join", "JoinStats": "join", "Tile": "join", "plan_batches": "join",
    "tensor_join": "join", "nlj_prefetch": "join", "tensor_join_vectors": "join",
    "join_prepared": "join", "join_embedded": "join", "e_selection": "join",
    "cosine_vm": "linalg", "top_k": "embedding",
    # models
    "EmbeddingModel": "embedding", "SyntheticModel": "embedding", "LookupModel": "embedding",
    "SubwordModel": "embedding", "embed_relation": "embedding",
    "embed_relation_device": "embedding", "prepare_relation": "embedding", "decode": "embedding",
    # device engine
    "prepare": "device", "PreparedRelation": "device",
    # matches file (cli._write_matches), formatted on the GPU
    "write_matches": "matchio", "format_matches": "matchio",
    # cost model (cost.py), calibrated on the GPU
    "CostParams": "cost", "calibrate": "cost", "choose_plan": "cost",
    "estimate_tensor": "cost", "estimate_nlj_prefetch": "cost", "estimate_nlj_naive": "cost",
    "estimate_selection": "cost",
}


def __getattr__(name):
    mod = _LAZY.get(name)
    if mod is None:
        raise AttributeError(name)
    import importlib
    return getattr(importlib.import_module(f".{mod}", __name__), name)


__all__ = sorted([
    "EmbeddedRelation", "MatchSet", "MatchSink", "RawRelation", "Threshold", "canonicalize",
    "make_raw_relation", "BudgetTooSmall", "BufferTooSmall", "CapacityExceeded",
    "DimensionMismatch", "OffsetOutOfRange", "OutOfVocabulary", "ParseError", "SimjoinError",
    "ZeroVector", *_LAZY])
