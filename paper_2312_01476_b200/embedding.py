"""Embedding models (mu) and the prefetch operator.

The model protocol is the reference's (embedding.py:32-69): ``dim``,
``latency_ns``, an exact lock-protected ``call_count``, ``embed(token)`` and
the batch hook ``_embed_into(tokens, out)``.  One hook is added for the GPU
path, ``_embed_into_device(tokens, out)``, filling a CUDA tensor; models whose
recipe runs on the GPU override it (SyntheticModel, LookupModel,
SubwordModel), the base implementation embeds on the host and copies.  Every
path counts exactly one model call per tuple, so prefetching touches mu
|R| + |S| times.
"""

from __future__ import annotations

import math
import threading
import time
from typing import Dict, Optional, Sequence

import os

import numpy as np
import torch

from . import device as D
from .core import EmbeddedRelation, RawRelation
from .errors import OffsetOutOfRange, OutOfVocabulary

_U64 = (1 << 64) - 1
_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def fnv1a64(data: bytes) -> int:
    """FNV-1a 64-bit (offset 0xcbf29ce484222325, prime 0x100000001b3)."""
    h = 0xCBF29CE484222325
    for b in data:
        h = ((h ^ b) * 0x100000001B3) & _U64
    return h


def _normalize_row_host(row: np.ndarray) -> None:
    """Host twin of the normalisation rule (sequential fp64 sum of squares,
    zero-row repair, fp64 divide) for single-token embed() calls."""
    r64 = row.astype(np.float64)
    ss = float(np.cumsum(r64 * r64)[-1]) if row.size else 0.0
    norm = math.sqrt(ss)
    if norm < 1e-12:
        row[0] = np.float32(1.0)
        r64 = row.astype(np.float64)
        norm = math.sqrt(float(np.cumsum(r64 * r64)[-1]))
    row[:] = (row.astype(np.float64) / norm).astype(np.float32)


def synthetic_vector(stream_seed: int, dim: int) -> np.ndarray:
    """One synthetic-model row on the host (splitmix64 stream, fp64 map to
    [-1, 1), fp32 truncation, normalisation) -- single-token path."""
    k = np.arange(1, dim + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(stream_seed & _U64) + k * _GAMMA
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    out = ((z.astype(np.float64) * 2.0 ** -64) * 2.0 - 1.0).astype(np.float32)
    _normalize_row_host(out)
    return out


def _busy_wait(ns: int) -> None:
    deadline = time.perf_counter_ns() + ns
    while time.perf_counter_ns() < deadline:
        pass


def _device(dev) -> torch.device:
    if dev is None:
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device(dev)


class EmbeddingModel:
    """Deterministic token -> fp32 vector with exact call accounting."""

    kind = "abstract"

    def __init__(self, dim: int, latency_ns: int = 0):
        if dim <= 0:
            raise ValueError(f"dim must be positive, got {dim}")
        if latency_ns < 0:
            raise ValueError("latency_ns must be >= 0")
        self.dim = dim
        self.latency_ns = latency_ns
        self._calls = 0
        self._lock = threading.Lock()

    @property
    def call_count(self) -> int:
        with self._lock:
            return self._calls

    def _count(self, n: int = 1) -> None:
        with self._lock:
            self._calls += n

    def _vector(self, token: str) -> np.ndarray:
        raise NotImplementedError

    def embed(self, token: str) -> np.ndarray:
        """One token, one model invocation."""
        vec = self._vector(token)
        self._count()
        if self.latency_ns:
            _busy_wait(self.latency_ns)
        return vec

    def _embed_into(self, tokens: Sequence[str], out: np.ndarray) -> None:
        for i, token in enumerate(tokens):
            out[i] = self.embed(token)

    def _embed_into_device(self, tokens: Sequence[str], out: torch.Tensor) -> None:
        """Fill the (n, dim) fp32 CUDA tensor `out`.  Default: host batch hook
        plus one host->device copy; GPU-native models override this."""
        host = np.empty((len(tokens), self.dim), dtype=np.float32)
        self._embed_into(tokens, host)
        out.copy_(torch.from_numpy(host))


class SyntheticModel(EmbeddingModel):
    """Reproducible pseudo-random unit vectors (embedding.py:72-107): stream
    seed = FNV-1a-64(utf-8 token) XOR model seed; splitmix64 components mapped
    to [-1, 1); normalised.  GPU batch path: fnv1a64 + synthetic_fill kernels."""

    kind = "synthetic"

    def __init__(self, dim: int, seed: int = 0, latency_ns: int = 0):
        super().__init__(dim, latency_ns)
        self.seed = seed & _U64

    def _stream_seed(self, token: str) -> int:
        return fnv1a64(token.encode("utf-8")) ^ self.seed

    def _vector(self, token: str) -> np.ndarray:
        return synthetic_vector(self._stream_seed(token), self.dim)

    def _embed_into(self, tokens: Sequence[str], out: np.ndarray) -> None:
        if self.latency_ns or len(tokens) == 0 or not torch.cuda.is_available():
            super()._embed_into(tokens, out)
            return
        dev = _device(None)
        t = torch.empty((len(tokens), self.dim), dtype=torch.float32, device=dev)
        self._embed_into_device(tokens, t)
        out[:] = t.cpu().numpy()

    def _embed_into_device(self, tokens: Sequence[str], out: torch.Tensor) -> None:
        if self.latency_ns:
            super()._embed_into_device(tokens, out)
            return
        if len(tokens):
            seeds = D.fnv1a64_tokens(tokens, self.seed, out.device)
            out.copy_(D.synthetic_rows(seeds, self.dim))
        self._count(len(tokens))


class LookupModel(EmbeddingModel):
    """Table-backed model (embedding.py:110-152).  OOV policy 'error' raises
    OutOfVocabulary; 'synthetic' falls back to the synthetic recipe.  The GPU
    path keeps the table resident on the device and gathers rows by index."""

    kind = "lookup"

    def __init__(self, table: Dict[str, np.ndarray], dim: int, oov: str = "error",
                 seed: int = 0, latency_ns: int = 0):
        super().__init__(dim, latency_ns)
        if oov not in ("error", "synthetic"):
            raise ValueError(f"unknown OOV policy {oov!r}")
        self.oov = oov
        self.seed = seed & _U64
        self._index: Dict[str, int] = {}
        rows = []
        for token, vec in table.items():
            arr = np.ascontiguousarray(vec, dtype=np.float32)
            if arr.shape != (dim,):
                raise ValueError(f"vector for {token!r} has shape {arr.shape}, want ({dim},)")
            if token in self._index:
                rows[self._index[token]] = arr
            else:
                self._index[token] = len(rows)
                rows.append(arr)
        self._matrix = (np.stack(rows) if rows else np.empty((0, dim), dtype=np.float32))
        self._matrix.flags.writeable = False
        self._dev_tables: Dict[torch.device, torch.Tensor] = {}

    @classmethod
    def from_matrix(cls, tokens: Sequence[str], matrix: np.ndarray, **kw) -> "LookupModel":
        m = cls({}, matrix.shape[1], **kw)
        m._index = {t: i for i, t in enumerate(tokens)}
        m._matrix = np.ascontiguousarray(matrix, dtype=np.float32)
        m._matrix.flags.writeable = False
        return m

    def __contains__(self, token: str) -> bool:
        return token in self._index

    def __len__(self) -> int:
        return len(self._index)

    def _vector(self, token: str) -> np.ndarray:
        i = self._index.get(token)
        if i is not None:
            return self._matrix[i].copy()
        if self.oov == "error":
            raise OutOfVocabulary(token)
        return synthetic_vector(fnv1a64(token.encode("utf-8")) ^ self.seed, self.dim)

    def device_table(self, dev: torch.device) -> torch.Tensor:
        t = self._dev_tables.get(dev)
        if t is None:
            t = torch.from_numpy(self._matrix.copy()).to(dev) if len(self._matrix) else \
                torch.zeros((1, self.dim), dtype=torch.float32, device=dev)
            self._dev_tables[dev] = t
        return t

    LOOKUP_THREADS = int(os.environ.get("SJB_LOOKUP_THREADS", str(min(16, os.cpu_count() or 1))))

    def indices(self, tokens: Sequence[str]) -> np.ndarray:
        """Table row of every token (-1 for OOV under the synthetic policy).
        With the native helper (csrc/sjb_pack.c): a C hash table of the
        vocabulary, built once, probed by several threads without the GIL;
        tokens that are not compact-ASCII str objects go through the dict.
        Without it, the same dict probes in Python (host marshalling only)."""
        try:
            from . import _sjbpack
            if getattr(self, "_cindex", None) is None:
                self._cindex = _sjbpack.build_index(self._index)
            idx = np.frombuffer(_sjbpack.lookup_mt(self._cindex, tokens, self.LOOKUP_THREADS),
                                dtype=np.int64)
            rest = np.nonzero(idx == -2)[0]
            if len(rest):
                get = self._index.get
                idx[rest] = [get(tokens[int(i)], -1) for i in rest]
        except (ImportError, AttributeError):
            get = self._index.get
            idx = np.fromiter((get(t, -1) for t in tokens), dtype=np.int64, count=len(tokens))
        if self.oov == "error" and len(idx) and idx.min() < 0:
            raise OutOfVocabulary(tokens[int(np.argmin(idx))])
        return idx

    def _embed_into_device(self, tokens: Sequence[str], out: torch.Tensor) -> None:
        if self.latency_ns:
            super()._embed_into_device(tokens, out)
            return
        idx = self.indices(tokens)
        dev = out.device
        oov = np.nonzero(idx < 0)[0]
        if len(idx):
            table = self.device_table(dev)
            safe = np.where(idx < 0, 0, idx)
            out.copy_(table.index_select(0, torch.from_numpy(safe).to(dev)))
            if len(oov):
                seeds = D.fnv1a64_tokens([tokens[i] for i in oov], self.seed, dev)
                out[torch.from_numpy(oov).to(dev)] = D.synthetic_rows(seeds, self.dim)
        self._count(len(tokens))


class SubwordModel(EmbeddingModel):
    """FastText-style subword model (BASELINE cfg3; no counterpart in the
    reference).  Row = mean of the bucket-table rows of the
    word hash and of every minn..maxn-gram of '<' token '>', bucket =
    FNV-1a-64(bytes) mod n_buckets, summed in fp32 in item order, divided by
    the item count.  Restated on the CPU in oracle/sj_oracle.c."""

    kind = "subword"

    def __init__(self, table, minn: int = 3, maxn: int = 6, latency_ns: int = 0):
        if isinstance(table, torch.Tensor):
            self._table_dev = table.contiguous()
            self._table_host = None
            dim = table.shape[1]
        else:
            self._table_host = np.ascontiguousarray(table, dtype=np.float32)
            self._table_dev = None
            dim = self._table_host.shape[1]
        super().__init__(dim, latency_ns)
        if minn < 1 or maxn < minn:
            raise ValueError("need 1 <= minn <= maxn")
        self.minn, self.maxn = minn, maxn

    @property
    def n_buckets(self) -> int:
        t = self._table_dev if self._table_dev is not None else self._table_host
        return int(t.shape[0])

    def table_on(self, dev: torch.device) -> torch.Tensor:
        if self._table_dev is None or self._table_dev.device != dev:
            src = self._table_dev if self._table_dev is not None else torch.from_numpy(
                self._table_host)
            self._table_dev = src.to(dev)
        return self._table_dev

    def items(self, token: str):
        b = token.encode("utf-8")
        m = b"<" + b + b">"
        yield b
        for n in range(self.minn, self.maxn + 1):
            for s in range(0, len(m) - n + 1):
                yield m[s:s + n]

    def _vector(self, token: str) -> np.ndarray:
        table = self._table_host if self._table_host is not None else \
            self._table_dev.cpu().numpy()
        acc = np.zeros(self.dim, dtype=np.float32)
        count = 0
        for it in self.items(token):
            acc = acc + table[fnv1a64(it) % table.shape[0]]
            count += 1
        return (acc / np.float32(count)).astype(np.float32)

    def _embed_into_device(self, tokens: Sequence[str], out: torch.Tensor) -> None:
        if self.latency_ns:
            super()._embed_into_device(tokens, out)
            return
        if len(tokens):
            out.copy_(D.subword_rows(tokens, self.table_on(out.device), self.minn, self.maxn))
        self._count(len(tokens))

    def embed_prepared(self, tokens: Sequence[str], dev: torch.device, name: str = ""):
        """Prefetch fused with normalise-and-cast: one kernel per relation."""
        prep = D.subword_rows(tokens, self.table_on(dev), self.minn, self.maxn,
                              prepared=True, name=name)
        self._count(len(tokens))
        return prep


def embed_relation(model: EmbeddingModel, r: RawRelation) -> EmbeddedRelation:
    """Embed every tuple once, in offset order (embedding.py:155-163); the
    result is not normalised."""
    out = np.empty((len(r), model.dim), dtype=np.float32)
    model._embed_into(r.tokens, out)
    return EmbeddedRelation(out, model.dim, False, r.name)


def embed_relation_device(model: EmbeddingModel, r: RawRelation,
                          dev: Optional[torch.device] = None) -> torch.Tensor:
    """Device prefetch: (|R|, dim) fp32 CUDA tensor, exactly |R| model calls."""
    dev = _device(dev)
    out = torch.empty((len(r), model.dim), dtype=torch.float32, device=dev)
    model._embed_into_device(r.tokens, out)
    return out


def prepare_relation(model: EmbeddingModel, r: RawRelation,
                     dev: Optional[torch.device] = None) -> D.PreparedRelation:
    """Prefetch + normalise-and-cast, fused where the model allows it."""
    dev = _device(dev)
    if isinstance(model, SubwordModel) and not model.latency_ns:
        return model.embed_prepared(r.tokens, dev, r.name)
    if isinstance(model, LookupModel) and not model.latency_ns and model.oov == "error":
        idx = torch.from_numpy(model.indices(r.tokens)).to(dev)
        prep = D.prepare_gather(model.device_table(dev), idx, r.name) if len(r) else \
            D.prepare(torch.empty((0, model.dim), dtype=torch.float32, device=dev), r.name)
        model._count(len(r))
        return prep
    return D.prepare(embed_relation_device(model, r, dev), r.name)


def top_k(model: EmbeddingModel, er: EmbeddedRelation, raw: RawRelation, probe: str,
          k: int):
    """The k most cosine-similar tokens to the probe, ties broken by lower
    offset (reference embedding.py:218-231); cosines on the device."""
    from .linalg import cosine_vm
    if k < 1:
        raise ValueError("k must be >= 1")
    if len(er) != len(raw):
        raise ValueError("embedded and raw relations disagree on cardinality")
    probe_vec = model.embed(probe)
    sims = cosine_vm(probe_vec, er)
    order = np.argsort(-sims, kind="stable")[:k]
    return [(raw.tokens[i], float(sims[i])) for i in order]


def decode(r: RawRelation, offset: int) -> str:
    """Original token of a tuple offset (embedding.py:166-171)."""
    if not 0 <= offset < len(r):
        raise OffsetOutOfRange(f"offset {offset} outside relation of {len(r)}")
    return r.tokens[offset]
