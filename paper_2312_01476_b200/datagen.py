"""Seeded synthetic workloads for the BASELINE.json configs.

No public dataset is involved (the paper's Wikipedia/FastText data is not
available); every input is drawn from numpy's PCG64 ``default_rng(seed)`` in a
fixed order, so the oracle and the GPU path see the same arrays.

clustered(): cfg1/cfg2/cfg5 recipe -- C centroids ~ N(0, I) normalised; each
  vector = centroid[id] + sigma * N(0, I) / sqrt(d), renormalised; ids uniform
  (or Zipf(s) sizes for cfg4).  Left and right share the centroids.
strings(): cfg3 recipe -- lowercase a-z strings, length U[3, 12]; a fraction of
  the right relation are copies of left strings with 1-2 random edits.
"""

from __future__ import annotations

from typing import List, Optional, Tuple

import numpy as np


def _unit_rows(x: np.ndarray) -> np.ndarray:
    n = np.sqrt(np.einsum("ij,ij->i", x, x, dtype=np.float64))
    n[n == 0] = 1.0
    return (x / n[:, None].astype(x.dtype)).astype(np.float32)


def centroids(n_centroids: int, dim: int, rng: np.random.Generator) -> np.ndarray:
    return _unit_rows(rng.standard_normal((n_centroids, dim), dtype=np.float32))


def cluster_ids(n: int, n_centroids: int, rng: np.random.Generator,
                zipf: Optional[float] = None) -> np.ndarray:
    if zipf is None:
        return rng.integers(0, n_centroids, size=n)
    p = 1.0 / np.arange(1, n_centroids + 1, dtype=np.float64) ** zipf
    p /= p.sum()
    return rng.choice(n_centroids, size=n, p=p)


def clustered_rows(n: int, cents: np.ndarray, sigma: float, rng: np.random.Generator,
                   zipf: Optional[float] = None, chunk: int = 1 << 18) -> np.ndarray:
    """n rows around `cents`; generated in chunks to bound temporaries."""
    c, dim = cents.shape
    ids = cluster_ids(n, c, rng, zipf)
    out = np.empty((n, dim), dtype=np.float32)
    scale = np.float32(sigma / np.sqrt(dim))
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        noise = rng.standard_normal((e - s, dim), dtype=np.float32)
        out[s:e] = _unit_rows(cents[ids[s:e]] + scale * noise)
    return out


def clustered_pair(n_left: int, n_right: int, dim: int, n_centroids: int, sigma: float,
                   seed: int = 0, zipf: Optional[float] = None
                   ) -> Tuple[np.ndarray, np.ndarray]:
    """(left, right) fp32 matrices sharing one set of centroids."""
    rng = np.random.default_rng(seed)
    cents = centroids(n_centroids, dim, rng)
    left = clustered_rows(n_left, cents, sigma, rng, zipf)
    right = clustered_rows(n_right, cents, sigma, rng, zipf)
    return left, right


# BASELINE.json configs (shapes only; see DESIGN.md for what each stands for)
CONFIGS = {
    "cfg1": dict(n_left=10_000, n_right=10_000, dim=100, n_centroids=1_000, sigma=0.5,
                 theta=0.8, seed=0),
    "cfg2": dict(n_left=100_000, n_right=1_000_000, dim=100, n_centroids=10_000, sigma=0.5,
                 theta=0.8, seed=0),
    "cfg5": dict(n_left=200_000, n_right=200_000, dim=100, n_centroids=500, sigma=0.5,
                 theta=0.8, seed=0),
    # wide embeddings; the full 1M x 4M join is R-sharded over 8 GPUs
    "cfg4": dict(n_left=1_000_000, n_right=4_000_000, dim=768, n_centroids=50_000, sigma=0.6,
                 theta=0.75, seed=0, zipf=1.1, bf16=True),
}


def round_bf16(x: np.ndarray) -> np.ndarray:
    """fp32 values rounded to the nearest bf16 (ties to even), as fp32: the
    values a bf16 relation holds, exactly representable in fp32."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    r = (b + np.uint32(0x7FFF) + ((b >> np.uint32(16)) & np.uint32(1))) & np.uint32(0xFFFF0000)
    return r.view(np.float32)


def bf16_bits(x: np.ndarray) -> np.ndarray:
    """The bf16 bit patterns (u16) of bf16-exact fp32 values."""
    return (np.ascontiguousarray(x, dtype=np.float32).view(np.uint32) >> np.uint32(16)).astype(
        np.uint16)


def config_vectors(name: str, **over):
    """Inputs of a BASELINE config.  cfg4 is d = 768 *bf16* (BASELINE.json
    configs[3]): its rows are rounded to bf16 values (returned as fp32 arrays
    of bf16-exact values -- what the reference receives; the GPU path takes
    them as bf16 tensors, see bf16_bits).  bf16=False keeps fp32 rows."""
    c = dict(CONFIGS[name])
    bf = over.pop("bf16", c.pop("bf16", False))
    c.update(over)
    L, S = clustered_pair(c["n_left"], c["n_right"], c["dim"], c["n_centroids"], c["sigma"],
                          c["seed"], zipf=c.get("zipf"))
    if bf:
        L, S = round_bf16(L), round_bf16(S)
    c["bf16"] = bf
    return (L, S), c


_ALPHA = np.frombuffer(b"abcdefghijklmnopqrstuvwxyz", dtype=np.uint8)


def _rand_word(rng: np.random.Generator, lo: int = 3, hi: int = 12) -> str:
    n = int(rng.integers(lo, hi + 1))
    return bytes(_ALPHA[rng.integers(0, 26, size=n)]).decode()


def _edit(w: str, rng: np.random.Generator) -> str:
    chars = list(w)
    for _ in range(int(rng.integers(1, 3))):
        op = int(rng.integers(0, 3))
        pos = int(rng.integers(0, len(chars) + (1 if op == 1 else 0)))
        c = chr(int(_ALPHA[rng.integers(0, 26)]))
        if op == 0 and chars:            # substitute
            chars[min(pos, len(chars) - 1)] = c
        elif op == 1:                    # insert
            chars.insert(pos, c)
        elif len(chars) > 1:             # delete
            del chars[min(pos, len(chars) - 1)]
    return "".join(chars)


def strings(n_left: int, n_right: int, shared_frac: float = 0.3, seed: int = 0
            ) -> Tuple[List[str], List[str]]:
    rng = np.random.default_rng(seed)
    left = [_rand_word(rng) for _ in range(n_left)]
    n_shared = int(round(shared_frac * n_right))
    src = rng.integers(0, max(1, n_left), size=n_shared)
    right = [_edit(left[int(i)], rng) for i in src] + \
            [_rand_word(rng) for _ in range(n_right - n_shared)]
    perm = rng.permutation(n_right)
    right = [right[int(i)] for i in perm]
    return left, right


def bucket_table(n_buckets: int, dim: int, seed: int = 0) -> np.ndarray:
    """cfg3 subword table ~ N(0, 1/dim) (host; the bench draws it on device)."""
    rng = np.random.default_rng(seed)
    return (rng.standard_normal((n_buckets, dim), dtype=np.float32)
            * np.float32(1.0 / np.sqrt(dim)))
