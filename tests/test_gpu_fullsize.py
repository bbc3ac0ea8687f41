"""BASELINE-size joins on the GPU, checked through properties that need no
full CPU join (the oracle would take hours at these sizes):

* canonical order: (left, right) strictly increasing, i.e. sorted and
  duplicate-free like MatchSet.canonicalize (core.py:196-213);
* every similarity >= fp32(theta) (the inclusive decision, linalg.py:151);
* complete rows: for a seeded sample of left rows, the GPU's matches of those
  rows (offsets, order and fp32 bits) equal the oracle's join of the sampled
  rows against the whole right relation;
* path agreement: the host-input public API (streamed S copy, split left,
  pinned result buffers) returns the same bits as the device-resident join,
  and R-sharded joins concatenate to it (multigpu's assembly rule).
"""
import os

import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu
THREADS = max(1, len(os.sched_getaffinity(0)))


def _check_canonical(lo, ro, so, theta):
    assert lo.dtype == np.uint64 and ro.dtype == np.uint64 and so.dtype == np.float32
    assert len(lo) == len(ro) == len(so)
    if len(lo) > 1:
        key_inc = (lo[1:] > lo[:-1]) | ((lo[1:] == lo[:-1]) & (ro[1:] > ro[:-1]))
        assert key_inc.all(), "not strictly increasing in (left, right)"
    assert (so >= np.float32(theta)).all()


def _rows_match_oracle(L, S, lo, ro, so, theta, n_rows, seed):
    rng = np.random.default_rng(seed)
    rows = np.sort(rng.choice(L.shape[0], size=n_rows, replace=False)).astype(np.uint64)
    wl, wr, ws = O.join_raw(L[rows.astype(np.int64)], S, theta, threads=THREADS)
    wl = rows[wl.astype(np.int64)]
    starts = np.searchsorted(lo, rows, side="left")
    ends = np.searchsorted(lo, rows, side="right")
    gl = np.concatenate([lo[a:b] for a, b in zip(starts, ends)])
    gr = np.concatenate([ro[a:b] for a, b in zip(starts, ends)])
    gs = np.concatenate([so[a:b] for a, b in zip(starts, ends)])
    assert len(wl) > 0, "sample without matches proves nothing"
    assert np.array_equal(gl, wl) and np.array_equal(gr, wr)
    assert np.array_equal(gs.view(np.uint32), ws.view(np.uint32))
    return len(wl)


def _device_join(L, S, theta):
    from paper_2312_01476_b200 import device as D
    dev = torch.device("cuda", 0)
    m = D.join_prepared(D.prepare(torch.from_numpy(L).to(dev)),
                        D.prepare(torch.from_numpy(S).to(dev)), theta)
    return m.to_host()


def test_cfg2_full_size():
    """BASELINE configs[1]: 100k x 1M, d = 100, theta = 0.8 (the bench workload)."""
    from paper_2312_01476_b200 import datagen
    from paper_2312_01476_b200 import multigpu as MG
    from paper_2312_01476_b200.join import tensor_join_vectors
    (L, S), c = datagen.config_vectors("cfg2")
    theta = c["theta"]
    lo, ro, so = _device_join(L, S, theta)
    _check_canonical(lo, ro, so, theta)
    assert len(lo) == 5_334_467           # the count every earlier run reported
    _rows_match_oracle(L, S, lo, ro, so, theta, 96, seed=1)
    # the public host-input path: streamed S copy, split left, pinned output
    ms, stats = tensor_join_vectors(torch.from_numpy(L).pin_memory(),
                                    torch.from_numpy(S).pin_memory(), theta,
                                    device=torch.device("cuda", 0))
    assert stats.pairs_compared == L.shape[0] * S.shape[0]
    assert np.array_equal(ms.lefts, lo) and np.array_equal(ms.rights, ro)
    assert np.array_equal(ms.sims.view(np.uint32), so.view(np.uint32))
    # R-sharded joins (3 ranks' row ranges on one device) concatenate to it
    dev = torch.device("cuda", 0)
    Sd = torch.from_numpy(S).to(dev)
    parts = []
    for r in range(3):
        r0, r1 = MG.shard_range(L.shape[0], r, 3)
        parts.append(MG.sharded_join_streamed(torch.from_numpy(L[r0:r1]).to(dev), Sd, theta, r0,
                                              chunks=4).to_host())
    cl, cr, cs = MG.concat_shards(parts)
    assert np.array_equal(cl, lo) and np.array_equal(cr, ro)
    assert np.array_equal(cs.view(np.uint32), so.view(np.uint32))


def test_cfg5_output_heavy_full_size():
    """BASELINE configs[4] at its most output-heavy threshold (8.1e7 matches:
    the deferred recheck, row bucketing and large-row sorts)."""
    from paper_2312_01476_b200 import datagen
    (L, S), c = datagen.config_vectors("cfg5")
    theta = 0.4
    lo, ro, so = _device_join(L, S, theta)
    _check_canonical(lo, ro, so, theta)
    assert len(lo) > 5e7
    _rows_match_oracle(L, S, lo, ro, so, theta, 64, seed=2)
    # a second run (deferred placement chosen from the first) is identical
    lo2, ro2, so2 = _device_join(L, S, theta)
    assert np.array_equal(lo2, lo) and np.array_equal(ro2, ro)
    assert np.array_equal(so2.view(np.uint32), so.view(np.uint32))


def test_cfg4_shape_wide():
    """BASELINE configs[3]'s distribution (d = 768, 50k centroids, sigma 0.6,
    Zipf(1.1) cluster sizes, theta = 0.75) at 20k x 400k: the wide filter and
    the tile-group recheck."""
    from paper_2312_01476_b200 import datagen
    (L, S), c = datagen.config_vectors("cfg4", n_left=20_000, n_right=400_000)
    theta = c["theta"]
    lo, ro, so = _device_join(L, S, theta)
    _check_canonical(lo, ro, so, theta)
    assert len(lo) > 1e7
    _rows_match_oracle(L, S, lo, ro, so, theta, 48, seed=3)
