"""Parity of the CUDA path with the reference (golden fixtures) and the
oracle.  Bar: bit-exact MatchSets (offsets, order, and fp32 similarity bits).
Every join here runs through libsjb200.so (tcgen05 filter + canonical recheck).
"""
import numpy as np
import pytest
import torch

import oracle as O
from conftest import case_inputs, golden_tokens

pytestmark = pytest.mark.gpu

GOLDEN_JOINS = ["c_small", "c_d4", "c_d64", "c_d16_neg", "c_one", "c_ragged", "c_all", "cfg1",
                "c_d200", "c_d768"]


def _bits_equal(ms, lo, ro, so):
    return (np.array_equal(ms.lefts, lo) and np.array_equal(ms.rights, ro)
            and np.array_equal(ms.sims.view(np.uint32), so.view(np.uint32)))


def _op_dtype(dim: int):
    """Operand image format: bf16 on the resident-R filter path (kpad <= 128),
    fp16 on the wide path (sjb_common.cuh op_is_bf16)."""
    from paper_2312_01476_b200 import device as D
    return torch.bfloat16 if D.kpad(dim) <= 128 else torch.float16


def _decode_operand(op: torch.Tensor, n: int, dim: int) -> np.ndarray:
    """Rebuild the row-major fp16 matrix from the tiled operand image."""
    from paper_2312_01476_b200 import device as D
    kpad = D.kpad(dim)
    a = op.view(torch.int16).cpu().numpy()
    T = 256
    tiles = a.size // (T * kpad)
    t = a.reshape(tiles, kpad // 8, T, 8).transpose(0, 2, 1, 3).reshape(tiles * T, kpad)
    return t[:n], t


@pytest.mark.parametrize("staged", [False, True])
@pytest.mark.parametrize("dim", [1, 3, 4, 16, 100, 128, 200, 768])
def test_normalize_and_operand_image(cuda, monkeypatch, dim, staged):
    """Bitwise sj_normalize_rows + the tiled operand image, through the
    pipelined kernel (dim % 4 == 0, kpad <= 128, aligned rows) and the staged
    one (every other case; SJB_PREP_STAGED forces it)."""
    from paper_2312_01476_b200 import device as D
    if staged:
        monkeypatch.setenv("SJB_PREP_STAGED", "1")
    rng = np.random.default_rng(dim)
    n = 300
    x = rng.standard_normal((n, dim), dtype=np.float32) * rng.uniform(0.01, 10, (n, 1)).astype(np.float32)
    x[5] = 0.0
    x[17] = 1e-20
    x[23, ::2] = -0.0                    # signed zeros survive the quotient
    x[29, : (dim + 1) // 2] = 3.0e38     # huge and denormal magnitudes
    x[31] = np.float32(1e-44) * np.arange(1, dim + 1, dtype=np.float32)
    p = D.prepare(torch.from_numpy(x).to(cuda))
    want, rep = O.normalize_rows(x)
    assert np.array_equal(p.f32.cpu().numpy().view(np.uint32), want.view(np.uint32))
    assert p.repaired() == rep and rep >= 2   # rows 5, 17 (+ 23, 31 when dim is tiny)
    # input rows 4 bytes off 16-byte alignment: the scalar staging path
    buf = torch.empty(n * dim + 1, device=cuda)
    xs = buf[1:].view(n, dim)
    xs.copy_(torch.from_numpy(x))
    q = D.prepare(xs)
    assert np.array_equal(q.f32.cpu().numpy().view(np.uint32), want.view(np.uint32))
    rows, full = _decode_operand(p.op, n, dim)
    bf = torch.from_numpy(want).to(_op_dtype(dim)).view(torch.int16).numpy()
    kpad = full.shape[1]
    assert np.array_equal(rows[:, :dim], bf)
    assert (rows[:, dim:] == 0).all() and (full[n:] == 0).all()
    assert full.shape[0] % 256 == 0 and kpad % 16 == 0
    assert kpad == (dim + 15) // 16 * 16 if dim <= 128 else kpad == (dim + 63) // 64 * 64


@pytest.mark.parametrize("name", GOLDEN_JOINS)
def test_golden_tensor_join_public_api(cuda, golden, manifest, name):
    from paper_2312_01476_b200 import LookupModel, RawRelation, tensor_join
    meta = manifest["cases"][name]
    L, S = case_inputs(meta)
    toks_l = [f"L{i}" for i in range(len(L))]
    toks_r = [f"S{i}" for i in range(len(S))]
    model = LookupModel.from_matrix(toks_l + toks_r, np.concatenate([L, S]))
    ms, st = tensor_join(RawRelation("left", toks_l), RawRelation("right", toks_r), model,
                         meta["theta"], budget_bytes=64 << 20, threads=8)
    assert _bits_equal(ms, golden[name + "_l"], golden[name + "_r"], golden[name + "_s"])
    assert st.matches == meta["matches"] == len(ms)
    assert st.model_calls_left == len(L) and st.model_calls_right == len(S)
    assert model.call_count == len(L) + len(S)
    assert st.pairs_compared == len(L) * len(S) and st.algo == "tensor"


@pytest.mark.parametrize("name", ["c_small", "c_d64", "cfg1"])
def test_golden_vectors_api(cuda, golden, manifest, name):
    from paper_2312_01476_b200.join import tensor_join_vectors
    meta = manifest["cases"][name]
    L, S = case_inputs(meta)
    ms, _ = tensor_join_vectors(L, S, meta["theta"])
    assert _bits_equal(ms, golden[name + "_l"], golden[name + "_r"], golden[name + "_s"])


def test_synthetic_model_on_device(cuda, golden):
    from paper_2312_01476_b200 import RawRelation, SyntheticModel, embed_relation_device
    toks = golden_tokens(golden)
    for dim, seed in ((16, 7), (4, 1), (100, 0)):
        m = SyntheticModel(dim, seed=seed)
        v = embed_relation_device(m, RawRelation("x", toks)).cpu().numpy()
        assert np.array_equal(v.view(np.uint32), golden[f"syn_{dim}_{seed}"].view(np.uint32))
        assert m.call_count == len(toks)


@pytest.mark.parametrize("theta", [0.0, 0.3, -1.0])
def test_synthetic_join_and_nlj(cuda, golden, small_relations, theta):
    from paper_2312_01476_b200 import SyntheticModel, nlj_prefetch, tensor_join
    left, right = small_relations
    model = SyntheticModel(16, seed=7)
    ms, st = tensor_join(left, right, model, theta, budget_bytes=4096)
    k = f"synjoin_{theta}"
    assert _bits_equal(ms, golden[k + "_l"], golden[k + "_r"], golden[k + "_s"])
    ms2, st2 = nlj_prefetch(left, right, model, theta, threads=4)
    assert ms2 == ms
    assert st2.inner_relation == "right" and st2.algo == "prefetch_nlj"
    assert model.call_count == 2 * (len(left) + len(right))


def test_random_instances_match_oracle(cuda):
    """SPEC acceptance (1)-style sweep: 50 seeded instances, all dims 1..128."""
    from paper_2312_01476_b200 import device as D
    rng = np.random.default_rng(2024)
    for inst in range(50):
        nl, nr = int(rng.integers(1, 700)), int(rng.integers(1, 700))
        dim = int(rng.integers(1, 129))
        c = int(rng.integers(1, 60))
        L, S = O_pair(nl, nr, dim, c, float(rng.uniform(0.2, 1.0)), inst)
        theta = float(rng.uniform(-0.2, 0.95))
        pl = D.prepare(torch.from_numpy(L).to(cuda))
        pr = D.prepare(torch.from_numpy(S).to(cuda))
        m = D.join_prepared(pl, pr, theta)
        lo, ro, so = m.to_host()
        wl, wr, ws = O.join_raw(L, S, theta, threads=4)
        assert np.array_equal(lo, wl) and np.array_equal(ro, wr), (inst, nl, nr, dim, theta)
        assert np.array_equal(so.view(np.uint32), ws.view(np.uint32)), inst


def test_random_wide_instances_match_oracle(cuda):
    """Wide embeddings (dim 129..800): the K-streaming filter kernel."""
    from paper_2312_01476_b200 import device as D
    rng = np.random.default_rng(4096)
    for inst in range(16):
        nl, nr = int(rng.integers(1, 600)), int(rng.integers(1, 900))
        dim = int(rng.integers(129, 801))
        c = int(rng.integers(1, 40))
        L, S = O_pair(nl, nr, dim, c, float(rng.uniform(0.3, 1.0)), 100 + inst)
        theta = float(rng.uniform(-0.1, 0.9))
        pl = D.prepare(torch.from_numpy(L).to(cuda))
        pr = D.prepare(torch.from_numpy(S).to(cuda))
        m = D.join_prepared(pl, pr, theta)
        lo, ro, so = m.to_host()
        wl, wr, ws = O.join_raw(L, S, theta, threads=4)
        assert np.array_equal(lo, wl) and np.array_equal(ro, wr), (inst, nl, nr, dim, theta)
        assert np.array_equal(so.view(np.uint32), ws.view(np.uint32)), inst


@pytest.mark.parametrize("variant", ["fused", "tile", "group"])
def test_wide_recheck_variants(cuda, manifest, golden, monkeypatch, variant):
    """All wide recheck variants are exact: fused warps, the per-tile staged
    kernel, and the tile-group kernel (default) that reuses the A chunks."""
    from paper_2312_01476_b200 import device as D
    if variant != "group":
        meta0 = manifest["cases"]["c_d200"]
        L0, S0 = case_inputs(meta0)
        if _ab_gate(D, monkeypatch, ("SJB_WIDE_RECHECK", variant), lambda: D.join_prepared(
                D.prepare(torch.from_numpy(L0).to(cuda)),
                D.prepare(torch.from_numpy(S0).to(cuda)), meta0["theta"])):
            return
    monkeypatch.setenv("SJB_WIDE_RECHECK", variant)
    for name in ("c_d200", "c_d768"):
        meta = manifest["cases"][name]
        L, S = case_inputs(meta)
        m = D.join_prepared(D.prepare(torch.from_numpy(L).to(cuda)),
                            D.prepare(torch.from_numpy(S).to(cuda)), meta["theta"])
        lo, ro, so = m.to_host()
        assert np.array_equal(lo, golden[name + "_l"]) and np.array_equal(ro, golden[name + "_r"])
        assert np.array_equal(so.view(np.uint32), golden[name + "_s"].view(np.uint32))


def test_wide_overflow_retry_and_all_pairs(cuda, manifest, golden):
    from paper_2312_01476_b200 import device as D
    meta = manifest["cases"]["c_d768"]
    L, S = case_inputs(meta)
    pl = D.prepare(torch.from_numpy(L).to(cuda))
    pr = D.prepare(torch.from_numpy(S).to(cuda))
    m = D.join_prepared(pl, pr, meta["theta"], cand_cap=64)   # forces the retry
    assert m.retries >= 1
    lo, ro, so = m.to_host()
    assert np.array_equal(lo, golden["c_d768_l"]) and np.array_equal(ro, golden["c_d768_r"])
    assert np.array_equal(so.view(np.uint32), golden["c_d768_s"].view(np.uint32))
    m = D.join_prepared(pl, pr, -1.0)
    lo, ro, so = m.to_host()
    assert len(lo) == len(L) * len(S)
    wl, wr, ws = O.join_raw(L, S, -1.0, threads=8)
    assert np.array_equal(lo, wl) and np.array_equal(ro, wr)
    assert np.array_equal(so.view(np.uint32), ws.view(np.uint32))


@pytest.mark.parametrize("staged", [False, True])
@pytest.mark.parametrize("dim", [3, 100, 768])
def test_rounding_error_outputs(cuda, dim, monkeypatch, staged):
    """row_err bounds ||op16(x) - x|| from above (tightly); tile_err is the
    per-256-row-tile maximum (zero for padding tiles)."""
    from paper_2312_01476_b200 import device as D
    if staged:
        monkeypatch.setenv("SJB_PREP_STAGED", "1")
    rng = np.random.default_rng(dim + 5)
    n = 700
    x = rng.standard_normal((n, dim), dtype=np.float32)
    x[9] = 0.0
    p = D.prepare(torch.from_numpy(x).to(cuda))
    f = p.f32.cpu().numpy()
    bf = torch.from_numpy(f).to(_op_dtype(dim)).to(torch.float64).numpy()
    want = np.sqrt(((bf - f.astype(np.float64)) ** 2).sum(axis=1))
    got = p.row_err.cpu().numpy().astype(np.float64)[:n]
    assert (got >= want).all() and (got <= want * (1 + 1e-4) + 1e-30).all()
    tiles = p.tile_err.cpu().numpy()
    assert len(tiles) == D.tile_count(n)
    for t in range(len(tiles)):
        seg = got[t * 256:(t + 1) * 256]
        assert tiles[t] == (np.float32(seg.max()) if len(seg) else 0.0)


def test_per_row_band_is_exact_and_tighter(cuda, manifest, golden):
    """Same MatchSet with the per-row band as with the uniform one, fewer
    candidates: cfg1 (golden) and cfg4-shaped wide data (oracle)."""
    from paper_2312_01476_b200 import datagen, device as D
    meta = manifest["cases"]["cfg1"]
    L, S = case_inputs(meta)
    wide = datagen.clustered_pair(500, 900, 768, 40, 0.6, 3, zipf=1.1)
    wl, wr, ws = O.join_raw(wide[0], wide[1], 0.75, threads=8)
    cases = [(L, S, meta["theta"], golden["cfg1_l"], golden["cfg1_r"], golden["cfg1_s"]),
             (wide[0], wide[1], 0.75, wl, wr, ws)]
    for L, S, theta, el, er, es in cases:
        pl = D.prepare(torch.from_numpy(L).to(cuda))
        pr = D.prepare(torch.from_numpy(S).to(cuda))
        a = D.join_prepared(pl, pr, theta, per_row_band=True)
        b = D.join_prepared(pl, pr, theta, per_row_band=False)
        for m in (a, b):
            lo, ro, so = m.to_host()
            assert np.array_equal(lo, el) and np.array_equal(ro, er)
            assert np.array_equal(so.view(np.uint32), es.view(np.uint32))
        assert a.n_candidates < b.n_candidates, (L.shape, a.n_candidates, b.n_candidates)


@pytest.mark.parametrize("chunks", [1, 3, 8])
@pytest.mark.parametrize("pinned", [True, False])
def test_streamed_join_matches_golden(cuda, manifest, golden, chunks, pinned):
    """S copied in chunks and filtered per S-tile range (sjb_join_begin /
    filter_tiles / finish): identical MatchSet."""
    from paper_2312_01476_b200 import device as D
    for name in ("cfg1", "c_ragged", "c_d768"):
        meta = manifest["cases"][name]
        L, S = case_inputs(meta)
        Sh = torch.from_numpy(S)
        if pinned:
            Sh = Sh.pin_memory()
        m, R = D.join_streamed(D.prepare(torch.from_numpy(L).to(cuda)), Sh, meta["theta"],
                               chunks=chunks)
        lo, ro, so = m.to_host()
        assert np.array_equal(lo, golden[name + "_l"]) and np.array_equal(ro, golden[name + "_r"])
        assert np.array_equal(so.view(np.uint32), golden[name + "_s"].view(np.uint32))
        ref = D.prepare(torch.from_numpy(S).to(cuda))
        assert torch.equal(R.f32, ref.f32) and torch.equal(R.op.view(torch.int16), ref.op.view(torch.int16))
        assert torch.equal(R.row_err[:R.n], ref.row_err[:R.n])


def test_streamed_join_overflow_and_vectors_api(cuda, manifest, golden):
    from paper_2312_01476_b200 import device as D
    from paper_2312_01476_b200.join import tensor_join_vectors
    import paper_2312_01476_b200.join as J
    meta = manifest["cases"]["cfg1"]
    L, S = case_inputs(meta)
    D._cap_cache.clear()
    old = D.initial_capacity
    D.initial_capacity = lambda a, b: 1000           # force the overflow retry
    try:
        m, _ = D.join_streamed(D.prepare(torch.from_numpy(L).to(cuda)), torch.from_numpy(S),
                               meta["theta"], chunks=4)
    finally:
        D.initial_capacity = old
        D._cap_cache.clear()
    assert m.retries == 1
    lo, ro, so = m.to_host()
    assert np.array_equal(lo, golden["cfg1_l"]) and np.array_equal(so.view(np.uint32), golden["cfg1_s"].view(np.uint32))
    old_min = J._STREAM_MIN_ROWS
    J._STREAM_MIN_ROWS = 1                            # route through the streamed path
    try:
        ms, st = tensor_join_vectors(L, S, meta["theta"])
    finally:
        J._STREAM_MIN_ROWS = old_min
    assert np.array_equal(ms.lefts, golden["cfg1_l"]) and np.array_equal(ms.rights, golden["cfg1_r"])
    assert st.pairs_compared == len(L) * len(S)


def test_sharded_join_streamed_single_rank(cuda, manifest, golden):
    """The streamed R-sharded join (chunked S broadcast + per-chunk filter) on
    one rank: two shards joined separately concatenate to the golden set."""
    from paper_2312_01476_b200 import multigpu as MG
    meta = manifest["cases"]["cfg1"]
    L, S = case_inputs(meta)
    Sd = torch.from_numpy(S).to(cuda)
    S0 = Sd.clone()
    parts = []
    for r in range(2):
        r0, r1 = MG.shard_range(len(L), r, 2)
        m = MG.sharded_join_streamed(torch.from_numpy(L[r0:r1]).to(cuda), Sd, meta["theta"], r0,
                                     chunks=5)
        parts.append(m.to_host())
    assert torch.equal(Sd, S0)                  # the source S is left unchanged
    lo, ro, so = MG.concat_shards(parts)
    assert np.array_equal(lo, golden["cfg1_l"]) and np.array_equal(ro, golden["cfg1_r"])
    assert np.array_equal(so.view(np.uint32), golden["cfg1_s"].view(np.uint32))


@pytest.mark.parametrize("rounds,grid", [(1, 0), (4, 132), (0, 100)])
def test_owner_prepared_join_single_rank(cuda, manifest, golden, rounds, grid):
    """multigpu.sharded_join_owned on one rank: S prepared piece by piece into
    padded buffers (device.prepare_into), filtered round by round
    (device.JoinSession) on a reduced grid (SMs left to NCCL) -- the golden
    set, and a prepared S bitwise equal to a one-shot prepare."""
    from paper_2312_01476_b200 import device as D
    from paper_2312_01476_b200 import multigpu as MG
    meta = manifest["cases"]["cfg1"]
    L, S = case_inputs(meta)
    lay = MG.piece_layout(len(S), 1, rounds)
    assert lay.rounds == (rounds or lay.rounds) and lay.rows >= len(S)
    S_loc = torch.from_numpy(MG.local_pieces(S, lay, 0)).to(cuda)
    m, PR = MG.sharded_join_owned(torch.from_numpy(L).to(cuda), S_loc, lay, meta["theta"], 0,
                                  ops=MG.DeviceOps(grid=grid))
    lo, ro, so = m.to_host()
    assert np.array_equal(lo, golden["cfg1_l"]) and np.array_equal(ro, golden["cfg1_r"])
    assert np.array_equal(so.view(np.uint32), golden["cfg1_s"].view(np.uint32))
    ref = D.prepare(torch.from_numpy(S).to(cuda))
    n = len(S)
    assert torch.equal(PR.f32[:n], ref.f32)
    assert torch.equal(PR.op[:ref.op.numel()].view(torch.int16), ref.op.view(torch.int16))
    assert torch.equal(PR.row_err[:n], ref.row_err[:n])
    assert torch.equal(PR.tile_err[:D.tile_count(n)], ref.tile_err[:D.tile_count(n)])


def test_tensor_join_devices(cuda, manifest, golden):
    """tensor_join(devices=[...]): left rows sharded over devices (here two
    shards on the one GPU), S prepared once and copied; same MatchSet and
    model-call accounting as the single-device operator."""
    from paper_2312_01476_b200 import LookupModel, RawRelation, nlj_prefetch, tensor_join
    meta = manifest["cases"]["cfg1"]
    L, S = case_inputs(meta)
    toks_l = [f"L{i}" for i in range(len(L))]
    toks_r = [f"S{i}" for i in range(len(S))]
    model = LookupModel.from_matrix(toks_l + toks_r, np.concatenate([L, S]))
    for op in (tensor_join, nlj_prefetch):
        before = model.call_count
        args = (64 << 20,) if op is tensor_join else ()
        ms, st = op(RawRelation("left", toks_l), RawRelation("right", toks_r), model,
                    meta["theta"], *args, devices=[cuda, cuda, cuda])
        assert _bits_equal(ms, golden["cfg1_l"], golden["cfg1_r"], golden["cfg1_s"])
        assert model.call_count - before == len(L) + len(S)
        assert st.pairs_compared == len(L) * len(S) and st.matches == len(ms)


def _set_recheck(monkeypatch, recheck):
    """fused | deferred (cluster-blocked rows: dense blocks share staged S
    rows, sparse blocks per candidate) | deferred-grouped (the per-lane
    gather kernel: the dim % 4 != 0 fallback, and the A/B baseline)."""
    monkeypatch.setenv("SJB_RECHECK", recheck.split("-")[0])
    if "-" in recheck:
        monkeypatch.setenv("SJB_DENSE_RECHECK", recheck.split("-")[1])
    else:
        monkeypatch.delenv("SJB_DENSE_RECHECK", raising=False)


@pytest.mark.parametrize("recheck", ["fused", "deferred", "deferred-grouped"])
def test_recheck_placements(cuda, manifest, golden, monkeypatch, recheck):
    """d <= 128: fused recheck warps and the deferred full-occupancy kernels
    give the same bits (golden cases, overflow retry, theta = -1)."""
    from paper_2312_01476_b200 import device as D
    _set_recheck(monkeypatch, recheck)
    for name in ("cfg1", "c_small", "c_all", "c_d16_neg"):
        meta = manifest["cases"][name]
        L, S = case_inputs(meta)
        pl = D.prepare(torch.from_numpy(L).to(cuda))
        pr = D.prepare(torch.from_numpy(S).to(cuda))
        for cap in (None, 300):      # 300: forces the overflow retry (>= grid)
            m = D.join_prepared(pl, pr, meta["theta"], cand_cap=cap)
            lo, ro, so = m.to_host()
            assert np.array_equal(lo, golden[name + "_l"]) and np.array_equal(ro, golden[name + "_r"])
            assert np.array_equal(so.view(np.uint32), golden[name + "_s"].view(np.uint32))


def test_dense_rows_variant(cuda, manifest, golden, monkeypatch):
    """A/B: the one-warp-per-sorted-row dense recheck (SJB_DENSE_RECHECK=rows,
    per-lane 1-D copies or tile::gather4 of the S rows) -- built only with
    -DSJB_AB_KERNELS=1; the default library must reject the switch."""
    from paper_2312_01476_b200 import device as D
    meta0 = manifest["cases"]["c_small"]
    L0, S0 = case_inputs(meta0)
    monkeypatch.setenv("SJB_RECHECK", "deferred")
    if _ab_gate(D, monkeypatch, ("SJB_DENSE_RECHECK", "rows"), lambda: D.join_prepared(
            D.prepare(torch.from_numpy(L0).to(cuda)), D.prepare(torch.from_numpy(S0).to(cuda)),
            meta0["theta"])):
        return
    monkeypatch.setenv("SJB_DENSE_RECHECK", "rows")
    for g4 in ("1", "0"):
        monkeypatch.setenv("SJB_ROWS_G4", g4)
        for name in ("cfg1", "c_small", "c_all", "c_d16_neg"):
            meta = manifest["cases"][name]
            L, S = case_inputs(meta)
            for cap in (None, 300):
                m = D.join_prepared(D.prepare(torch.from_numpy(L).to(cuda)),
                                    D.prepare(torch.from_numpy(S).to(cuda)), meta["theta"],
                                    cand_cap=cap)
                lo, ro, so = m.to_host()
                assert np.array_equal(lo, golden[name + "_l"]) and np.array_equal(ro, golden[name + "_r"])
                assert np.array_equal(so.view(np.uint32), golden[name + "_s"].view(np.uint32))


def _ab_gate(D, monkeypatch, variant, call):
    """The A/B kernels are built only with -DSJB_AB_KERNELS=1: in the default
    library their switch must fail loudly (no silent fallback)."""
    from paper_2312_01476_b200 import _lib
    if _lib.lib().sjb_ab_kernels():
        return False
    monkeypatch.setenv(*variant)
    with pytest.raises(_lib.SjbError, match="A/B kernel"):
        call()
    return True


@pytest.mark.parametrize("variant", [("SJB_FILTER", "ts"), ("SJB_FILTER", "pair"),
                                     ("SJB_RBLOCK", "512")])
def test_filter_variants(cuda, manifest, golden, monkeypatch, variant):
    """d <= 128 filter kernels kept for A/B (TS-mode R block in tensor memory,
    CTA pair, two-tile R block) give the reference's bits on the golden cases,
    with and without the overflow retry, under both recheck placements."""
    from paper_2312_01476_b200 import device as D
    meta0 = manifest["cases"]["c_small"]
    L0, S0 = case_inputs(meta0)
    if _ab_gate(D, monkeypatch, variant, lambda: D.join_prepared(
            D.prepare(torch.from_numpy(L0).to(cuda)), D.prepare(torch.from_numpy(S0).to(cuda)),
            meta0["theta"])):
        return
    monkeypatch.setenv(*variant)
    for recheck in ("fused", "deferred"):
        monkeypatch.setenv("SJB_RECHECK", recheck)
        for name in ("cfg1", "c_small", "c_all", "c_d16_neg"):
            meta = manifest["cases"][name]
            L, S = case_inputs(meta)
            pl = D.prepare(torch.from_numpy(L).to(cuda))
            pr = D.prepare(torch.from_numpy(S).to(cuda))
            for cap in (None, 300):
                m = D.join_prepared(pl, pr, meta["theta"], cand_cap=cap)
                lo, ro, so = m.to_host()
                assert np.array_equal(lo, golden[name + "_l"]), (variant, recheck, name, cap)
                assert np.array_equal(ro, golden[name + "_r"]), (variant, recheck, name, cap)
                assert np.array_equal(so.view(np.uint32), golden[name + "_s"].view(np.uint32))


def test_cosine_vm_e_selection_top_k(cuda, golden, manifest):
    """sjb_cosine_vm and the operators on it against the reference's own
    outputs (e_selection join.py:145-179, top_k embedding.py:218-231)."""
    from paper_2312_01476_b200 import (EmbeddedRelation, RawRelation, SyntheticModel, ZeroVector,
                                       cosine_vm, e_selection, embed_relation, top_k)
    got = cosine_vm(golden["cos_vm_a"], EmbeddedRelation(golden["cos_vm_m"], 37, False, "c"))
    assert np.array_equal(got.view(np.uint32), golden["cos_vm_out"].view(np.uint32))
    rel = RawRelation("sel", [f"l_{i}" for i in range(40)] + ["dog", "cat", "été"])
    for th in (0.0, 0.2):
        model = SyntheticModel(16, seed=7)
        ms, st = e_selection(rel, model, "probe_word", th)
        k = f"esel_{th}"
        assert _bits_equal(ms, golden[k + "_l"], golden[k + "_r"], golden[k + "_s"])
        assert [st.model_calls_left, st.model_calls_right] == manifest["cases"][k]["model_calls"]
        assert model.call_count == len(rel) + 1 and st.algo == "e_selection"
    model = SyntheticModel(16, seed=7)
    tk = top_k(model, embed_relation(model, rel), rel, "probe_word", 7)
    assert [t for t, _ in tk] == [t for t, _ in manifest["top_k_probe_word_7"]]
    assert np.array_equal(np.array([s for _, s in tk], dtype=np.float32).view(np.uint32),
                          golden["top_k_sims"].view(np.uint32))
    with pytest.raises(ZeroVector):
        cosine_vm(np.zeros(37, np.float32), golden["cos_vm_m"])
    z = golden["cos_vm_m"].copy()
    z[5] = 0
    with pytest.raises(ZeroVector):
        cosine_vm(golden["cos_vm_a"], z)
    with pytest.raises(ValueError):
        top_k(model, embed_relation(model, rel), rel, "p", 0)


@pytest.mark.parametrize("recheck", ["fused", "deferred", "deferred-grouped"])
def test_medium_instances_match_oracle(cuda, monkeypatch, recheck):
    """Thousands of rows (several work items and S tiles per CTA, partial
    last tiles), dense and sparse thresholds, both recheck placements."""
    from paper_2312_01476_b200 import device as D
    _set_recheck(monkeypatch, recheck)
    rng = np.random.default_rng(77)
    for inst in range(4):
        nl, nr = int(rng.integers(3000, 7000)), int(rng.integers(4000, 9000))
        dim = int(rng.choice([37, 64, 100, 128]))
        L, S = O_pair(nl, nr, dim, int(rng.integers(20, 200)), float(rng.uniform(0.3, 0.8)),
                      500 + inst)
        theta = float(rng.choice([0.2, 0.5, 0.8, 0.95]))
        m = D.join_prepared(D.prepare(torch.from_numpy(L).to(cuda)),
                            D.prepare(torch.from_numpy(S).to(cuda)), theta)
        lo, ro, so = m.to_host()
        wl, wr, ws = O.join_raw(L, S, theta, threads=16)
        assert np.array_equal(lo, wl) and np.array_equal(ro, wr), (inst, nl, nr, dim, theta)
        assert np.array_equal(so.view(np.uint32), ws.view(np.uint32)), inst


@pytest.mark.parametrize("dim", [16, 64, 100, 128])
def test_dense_blocks_match_oracle(cuda, monkeypatch, dim):
    """The cluster-blocked dense recheck: clusters whose right members fit one
    staging window (~60), span several windows (~400) and approach the
    1024-row union cap (~900), plus a theta low enough for rows above the
    sortable 1024 candidates (sparse per-candidate blocks) -- every MatchSet
    equal to the oracle's, bit for bit."""
    from paper_2312_01476_b200 import device as D
    _set_recheck(monkeypatch, "deferred")
    cases = [(2000, 3000, 50, 0.3, 0.3), (1500, 4000, 10, 0.3, 0.3), (1200, 4500, 5, 0.3, 0.3),
             (700, 2600, 2, 0.6, -0.2)]
    for k, (nl, nr, c, sigma, theta) in enumerate(cases):
        L, S = O_pair(nl, nr, dim, c, sigma, 900 + k)
        m = D.join_prepared(D.prepare(torch.from_numpy(L).to(cuda)),
                            D.prepare(torch.from_numpy(S).to(cuda)), theta)
        lo, ro, so = m.to_host()
        wl, wr, ws = O.join_raw(L, S, theta, threads=16)
        assert len(wl) > 0
        assert np.array_equal(lo, wl) and np.array_equal(ro, wr), (dim, k)
        assert np.array_equal(so.view(np.uint32), ws.view(np.uint32)), (dim, k)


def test_dense_recheck_random_shapes(cuda, monkeypatch):
    """Deferred (dense) recheck on random small shapes: 1-row and 1-column
    relations, every dim % 4 == 0 up to 128 (and odd dims: the gather
    fallback), duplicate rows (equal similarities), zero rows (repaired),
    thetas from -0.3 to 0.95, and a tiny candidate capacity forcing the
    overflow retry -- each MatchSet bitwise the oracle's."""
    from paper_2312_01476_b200 import device as D
    _set_recheck(monkeypatch, "deferred")
    rng = np.random.default_rng(4242)
    for inst in range(24):
        nl = int(rng.choice([1, 2, 33, int(rng.integers(40, 2500))]))
        nr = int(rng.choice([1, 7, int(rng.integers(50, 4000))]))
        dim = int(rng.choice([4, 8, 16, 36, 64, 100, 128, 37, 101]))
        c = int(rng.integers(1, 60))
        L, S = O_pair(nl, nr, dim, c, float(rng.uniform(0.2, 0.8)), 7000 + inst)
        if nr > 10:
            S[3] = S[5]            # duplicate right rows
            S[7] = 0.0             # a zero row (repaired to e0)
        if nl > 10:
            L[2] = L[4]
        theta = float(rng.choice([-0.3, 0.0, 0.3, 0.6, 0.8, 0.95]))
        wl, wr, ws = O.join_raw(L, S, theta, threads=16)
        pl = D.prepare(torch.from_numpy(L).to(cuda))
        pr = D.prepare(torch.from_numpy(S).to(cuda))
        for cap in (None, 256):
            m = D.join_prepared(pl, pr, theta, cand_cap=cap)
            lo, ro, so = m.to_host()
            assert np.array_equal(lo, wl) and np.array_equal(ro, wr), (inst, nl, nr, dim, theta, cap)
            assert np.array_equal(so.view(np.uint32), ws.view(np.uint32)), (inst, cap)


def test_budget_and_thread_invariance(cuda, manifest, golden):
    """SPEC acceptance (4) + thread-count invariance: the
    MatchSet is identical for every budget and thread count (the device path
    never materialises a budget-sized buffer; both are validated only)."""
    from paper_2312_01476_b200 import LookupModel, RawRelation, nlj_prefetch, tensor_join
    meta = manifest["cases"]["c_ragged"]
    L, S = case_inputs(meta)
    tl = [f"L{i}" for i in range(len(L))]
    tr = [f"S{i}" for i in range(len(S))]
    model = LookupModel.from_matrix(tl + tr, np.concatenate([L, S]))
    results = []
    for budget in (1 << 30, 64 << 20, 16 << 20, 1 << 20, 4096):
        for threads in (1, 4):
            ms, st = tensor_join(RawRelation("l", tl), RawRelation("r", tr), model, meta["theta"],
                                 budget_bytes=budget, threads=threads)
            results.append(ms)
            assert st.threads == threads and st.peak_buffer_bytes == 0
    ms2, _ = nlj_prefetch(RawRelation("l", tl), RawRelation("r", tr), model, meta["theta"],
                          threads=3)
    for ms in results + [ms2]:
        assert _bits_equal(ms, golden["c_ragged_l"], golden["c_ragged_r"], golden["c_ragged_s"])


@pytest.mark.parametrize("dim,recheck", [(16, "fused"), (16, "deferred"), (16, "deferred-grouped"),
                                         (200, "fused")])
def test_nan_and_inf_rows(cuda, monkeypatch, dim, recheck):
    """Rows with NaN or +-Inf normalise to NaN rows (inf / inf) exactly as the
    reference's normalize_row; their similarities are NaN, so they match
    nothing -- the filter, the per-row band and the recheck must agree."""
    from paper_2312_01476_b200 import device as D
    _set_recheck(monkeypatch, recheck)
    rng = np.random.default_rng(dim)
    L = rng.standard_normal((300, dim)).astype(np.float32)
    S = rng.standard_normal((400, dim)).astype(np.float32)
    L[3, 2] = np.nan
    L[7, 0] = np.inf
    S[5, 1] = -np.inf
    S[9, :] = np.nan
    for theta in (-1.0, 0.1):
        pl, pr = D.prepare(torch.from_numpy(L).to(cuda)), D.prepare(torch.from_numpy(S).to(cuda))
        want32, _ = O.normalize_rows(L)
        assert np.array_equal(pl.f32.cpu().numpy().view(np.uint32), want32.view(np.uint32))
        lo, ro, so = D.join_prepared(pl, pr, theta).to_host()
        wl, wr, ws = O.join_raw(L, S, theta, threads=4)
        assert np.array_equal(lo, wl) and np.array_equal(ro, wr)
        assert np.array_equal(so.view(np.uint32), ws.view(np.uint32))
        assert not ({3, 7} & set(lo.tolist())) and not ({5, 9} & set(ro.tolist()))


def O_pair(nl, nr, dim, c, sigma, seed):
    from paper_2312_01476_b200 import datagen
    return datagen.clustered_pair(nl, nr, dim, c, sigma, seed)


def test_overflow_retry_is_exact(cuda, manifest, golden):
    from paper_2312_01476_b200 import device as D
    meta = manifest["cases"]["c_small"]
    L, S = case_inputs(meta)
    pl = D.prepare(torch.from_numpy(L).to(cuda))
    pr = D.prepare(torch.from_numpy(S).to(cuda))
    m = D.join_prepared(pl, pr, meta["theta"], cand_cap=16)   # forces the retry
    assert m.retries >= 1
    lo, ro, so = m.to_host()
    assert np.array_equal(lo, golden["c_small_l"]) and np.array_equal(ro, golden["c_small_r"])
    assert np.array_equal(so.view(np.uint32), golden["c_small_s"].view(np.uint32))


@pytest.mark.parametrize("nr,nl", [(3000, 3), (20000, 3), (70000, 3), (1_100_000, 1)])
def test_all_pairs_large_rows(cuda, nr, nl):
    """theta = -1: every pair matches; rows longer than the warp sort (1024)
    go to the CTA sort -- whole in shared memory up to 26624 keys, ranked
    through a shared-memory bitmap beyond (1.1M: two 2^20-offset windows)."""
    from paper_2312_01476_b200 import device as D
    rng = np.random.default_rng(5)
    L = rng.standard_normal((nl, 16), dtype=np.float32)
    S = rng.standard_normal((nr, 16), dtype=np.float32)
    m = D.join_prepared(D.prepare(torch.from_numpy(L).to(cuda)),
                        D.prepare(torch.from_numpy(S).to(cuda)), -1.0)
    lo, ro, so = m.to_host()
    assert len(lo) == nl * nr
    assert np.array_equal(lo, np.repeat(np.arange(nl, dtype=np.uint64), nr))
    assert np.array_equal(ro, np.tile(np.arange(nr, dtype=np.uint64), nl))
    Ln, _ = O.normalize_rows(L)
    Sn, _ = O.normalize_rows(S)
    for r in range(nl):
        assert np.array_equal(so[r * nr:(r + 1) * nr].view(np.uint32),
                              O.dots_vm(Ln[r], Sn).view(np.uint32))


def test_empty_and_errors(cuda):
    from paper_2312_01476_b200 import (BudgetTooSmall, DimensionMismatch, RawRelation,
                                       SyntheticModel, tensor_join, nlj_prefetch)
    from paper_2312_01476_b200.join import tensor_join_vectors
    m = SyntheticModel(8)
    e = RawRelation("e", [])
    r = RawRelation("r", ["a", "b"])
    ms, st = tensor_join(r, e, m, 0.5, budget_bytes=1024)
    assert len(ms) == 0 and st.pairs_compared == 0 and st.peak_buffer_bytes == 0
    ms, st = tensor_join(e, e, m, 0.5, budget_bytes=1024)
    assert len(ms) == 0
    with pytest.raises(ValueError):
        tensor_join(r, r, m, 0.5, budget_bytes=1024, threads=0)
    with pytest.raises(BudgetTooSmall):
        tensor_join(r, r, m, 0.5, budget_bytes=3)
    with pytest.raises(ValueError):
        nlj_prefetch(r, r, m, 1.5)
    with pytest.raises(DimensionMismatch):
        tensor_join_vectors(np.ones((2, 3), np.float32), np.ones((2, 4), np.float32), 0.1)


@pytest.mark.parametrize("dim,fused", [(100, False), (100, True), (200, False), (37, False)])
def test_subword_model_matches_oracle(cuda, monkeypatch, dim, fused):
    """Subword embedding on the GPU, bitwise the oracle's: the vectorised
    gather + normalise pass (dim % 4 == 0, <= 256), and the one-kernel
    fused path (SJB_SUBWORD_FUSED, or any other dim)."""
    from paper_2312_01476_b200 import RawRelation, SubwordModel, datagen, device as D
    from paper_2312_01476_b200.embedding import embed_relation_device, prepare_relation
    if fused:
        monkeypatch.setenv("SJB_SUBWORD_FUSED", "1")
    table = datagen.bucket_table(5003, dim, seed=1)
    left, right = datagen.strings(700, 900, seed=4)
    left += ["", "a", "ab", "abcdefghijklmnopqrstuvwxyzabcdefghijklmnop"]   # edge lengths
    m = SubwordModel(table)
    got = embed_relation_device(m, RawRelation("l", left)).cpu().numpy()
    want = O.subword_embed(left, table)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    pl = prepare_relation(m, RawRelation("l", left))      # fused embed+normalise+cast
    pr = prepare_relation(m, RawRelation("r", right))
    assert m.call_count == len(left) * 2 + len(right)
    wn, _ = O.normalize_rows(want)
    assert np.array_equal(pl.f32.cpu().numpy().view(np.uint32), wn.view(np.uint32))
    mm = D.join_prepared(pl, pr, 0.85)
    lo, ro, so = mm.to_host()
    wl, wr, ws = O.join_raw(want, O.subword_embed(right, table), 0.85)
    assert len(wl) > 0
    assert np.array_equal(lo, wl) and np.array_equal(ro, wr)
    assert np.array_equal(so.view(np.uint32), ws.view(np.uint32))


def test_cuda_kernel_backend(cuda, golden):
    from paper_2312_01476_b200 import kernels as K
    rng = np.random.default_rng(7)
    L = rng.standard_normal((70, 37), dtype=np.float32)
    S = rng.standard_normal((90, 37), dtype=np.float32)
    Ln, rep = O.normalize_rows(L)
    m = L.copy()
    assert K.normalize_rows_inplace(m) == rep
    assert np.array_equal(m.view(np.uint32), Ln.view(np.uint32))
    Sn, _ = O.normalize_rows(S)
    assert np.array_equal(K.row_norms(L).view(np.uint32), O.row_norms(L).view(np.uint32))
    bt = K.pack_transpose(Sn)
    assert np.array_equal(bt, Sn.T)
    out = np.empty((70, 90), np.float32)
    K.tile_dot(Ln, bt, out)
    assert np.array_equal(out.view(np.uint32), O.tile_dot(Ln, Sn).view(np.uint32))
    lo, ro, so = K.scan_hits(out, 0.1, 500, 7)
    ii, jj = np.nonzero(out >= np.float32(0.1))
    assert np.array_equal(lo, ii.astype(np.uint64) + 500)
    assert np.array_equal(ro, jj.astype(np.uint64) + 7)
    assert np.array_equal(so, out[ii, jj])
    assert np.array_equal(K.dots_vm(Ln[3], Sn).view(np.uint32), O.dots_vm(Ln[3], Sn).view(np.uint32))
    assert np.float32(K.dot_seq(Ln[1], Sn[2])) == O.dot_seq(Ln[1], Sn[2])
    chunks = K.nlj_rows(Ln, 10, 40, Sn, 0.2, 1e-4)
    wl, wr, ws = O.join_normalized(Ln[10:40], Sn, 0.2)
    assert np.array_equal(chunks[0][0], wl + 10) and np.array_equal(chunks[0][1], wr)
    toks = golden_tokens(golden)
    seeds = O.fnv1a64_many(toks, 7)
    v = np.empty((len(toks), 16), np.float32)
    K.synthetic_fill_many(seeds, v)
    assert np.array_equal(v.view(np.uint32), golden["syn_16_7"].view(np.uint32))


def _first_diff(a: bytes, b: bytes) -> str:
    i = next((k for k in range(min(len(a), len(b))) if a[k] != b[k]), min(len(a), len(b)))
    s = a.rfind(b"\n", 0, i) + 1
    return f"at byte {i}: got {a[s:s + 60]!r} want {b[s:s + 60]!r}"


def test_matches_file_bytes_match_reference_writer(cuda):
    """GPU matches file == the reference writer (cli.py:99-108, numpy per line)
    on probe floats (sweeps, powers of two, denormals, signs, inf/nan, -0) and
    u64 offsets of every decimal length."""
    import fmt_oracle as F
    from paper_2312_01476_b200.matchio import format_columns_device
    bits = F.probe_bits(60000, seed=1)
    bits = np.concatenate([bits, np.uint32([0, 0x80000000, 0x7F800000, 0xFF800000, 0x7FC00000])])
    n = bits.size
    rng = np.random.default_rng(5)
    lefts = (rng.random(n) * 10.0 ** rng.integers(0, 19, n)).astype(np.uint64)
    rights = rng.integers(0, 2**63, n, dtype=np.int64).astype(np.uint64) >> rng.integers(0, 63, n).astype(np.uint64)
    lefts[:3] = [0, 2**64 - 1, 10**19]
    sims = bits.view(np.float32)
    got = format_columns_device(torch.from_numpy(lefts.view(np.int64)).to(cuda),
                                torch.from_numpy(rights.view(np.int64)).to(cuda),
                                torch.from_numpy(sims).to(cuda)).cpu().numpy().tobytes()
    want = F.matches_file_reference(lefts, rights, sims)
    assert got == want, _first_diff(got, want)


def test_matches_file_of_a_join(cuda, tmp_path, manifest, golden):
    """write_matches of real join results (MatchSet and DeviceMatches), the
    empty result, and a 2M-line round trip."""
    import fmt_oracle as F
    from paper_2312_01476_b200 import MatchSet, device as D
    from paper_2312_01476_b200.matchio import format_matches, write_matches
    for name in ("c_small", "c_d16_neg", "cfg1"):
        lo, ro, so = golden[name + "_l"], golden[name + "_r"], golden[name + "_s"]
        ms = MatchSet("left", "right", lo, ro, so)
        p = tmp_path / f"{name}.csv"
        write_matches(str(p), ms)
        assert p.read_bytes() == F.matches_file_reference(lo, ro, so)
    meta = manifest["cases"]["cfg1"]
    L, S = case_inputs(meta)
    m = D.join_prepared(D.prepare(torch.from_numpy(L).to(cuda)),
                        D.prepare(torch.from_numpy(S).to(cuda)), meta["theta"])
    assert format_matches(m) == F.matches_file_reference(*m.to_host())
    write_matches(str(tmp_path / "empty.csv"), MatchSet("a", "b"))
    assert (tmp_path / "empty.csv").read_bytes() == b""
    # size-independent property at 2M lines: the file parses back to the columns
    n = 2_000_000
    rng = np.random.default_rng(9)
    lefts = np.sort(rng.integers(0, 10**6, n)).astype(np.uint64)
    rights = rng.integers(0, 4 * 10**6, n).astype(np.uint64)
    sims = rng.uniform(-1, 1, n).astype(np.float32)
    text = format_matches(MatchSet("a", "b", lefts, rights, sims))
    assert text.count(b"\n") == n and text.endswith(b"\n")
    cols = np.array(text.decode().replace("\n", ",").split(",")[:-1]).reshape(n, 3)
    assert np.array_equal(cols[:, 0].astype(np.uint64), lefts)
    assert np.array_equal(cols[:, 1].astype(np.uint64), rights)
    assert np.array_equal(cols[:, 2].astype(np.float64).astype(np.float32), sims)
    k = rng.integers(0, n, 20000)
    sub = F.matches_file_reference(lefts[k], rights[k], sims[k]).split(b"\n")[:-1]
    lines = text.split(b"\n")
    assert all(lines[i] == s for i, s in zip(k, sub))


def test_cost_calibration_on_device(cuda):
    """calibrate (cost.py:138-195) measured on the GPU: valid constants, and
    the plan choice routes BASELINE-sized joins to the tensor join."""
    from paper_2312_01476_b200 import SyntheticModel
    from paper_2312_01476_b200.cost import CostParams, calibrate, choose_plan
    model = SyntheticModel(100, seed=7)
    p = calibrate(model, 100, sample_sizes=(1000,))
    assert isinstance(p, CostParams) and 0.0 < p.tensor_efficiency < 1.0
    assert p.access_ns > 0 and p.model_ns > 0 and p.compare_per_dim_ns > 0
    assert model.call_count > 0
    for l, r in ((10_000, 10_000), (100_000, 1_000_000)):
        assert choose_plan(l, r, 100, 64 << 20, p)[0] == "tensor"
    with pytest.raises(ValueError):
        calibrate(model, 100, sample_sizes=(10,))


def test_host_split_join_with_overflowing_parts(cuda, monkeypatch):
    """The host-input join's pipelined parts (each queued before the previous
    part's count is read back) when every part overflows its first candidate
    capacity: the reruns are queued behind later parts and the result still
    equals the device-resident join, bit for bit."""
    from paper_2312_01476_b200 import device as D
    from paper_2312_01476_b200.join import _split_bounds, tensor_join_vectors
    rng = np.random.default_rng(11)
    cents = rng.standard_normal((40, 16)).astype(np.float32)
    L = (cents[rng.integers(0, 40, 32_768)] + 0.3 * rng.standard_normal((32_768, 16))).astype(np.float32)
    S = (cents[rng.integers(0, 40, 70_000)] + 0.3 * rng.standard_normal((70_000, 16))).astype(np.float32)
    theta = 0.9
    assert len(_split_bounds(L.shape[0])) == 4          # three parts
    ref = D.join_prepared(D.prepare(torch.from_numpy(L).to(cuda)),
                          D.prepare(torch.from_numpy(S).to(cuda)), theta).to_host()
    assert len(ref[0]) > 100_000
    monkeypatch.setattr(D, "initial_capacity", lambda nl, nr: 4096)
    monkeypatch.setattr(D, "_cap_cache", {})
    ms, _ = tensor_join_vectors(torch.from_numpy(L).pin_memory(), torch.from_numpy(S).pin_memory(),
                                theta, device=cuda)
    assert np.array_equal(ms.lefts, ref[0]) and np.array_equal(ms.rights, ref[1])
    assert np.array_equal(ms.sims.view(np.uint32), ref[2].view(np.uint32))


@pytest.mark.parametrize("left_kind", ["device", "numpy", "pinned"])
def test_host_input_join_input_kinds(cuda, left_kind):
    """tensor_join_vectors with a host right relation large enough to stream
    (>= 64k rows) and the left relation on the device, in pageable numpy
    memory or pinned: the staged copies, the split left preparation and the
    pipelined parts give the device join's bits."""
    from paper_2312_01476_b200 import device as D
    from paper_2312_01476_b200.join import tensor_join_vectors
    L, S = datagen_pair(20_480, 66_000, 24, seed=5)
    theta = 0.85
    ref = D.join_prepared(D.prepare(torch.from_numpy(L).to(cuda)),
                          D.prepare(torch.from_numpy(S).to(cuda)), theta).to_host()
    assert len(ref[0]) > 10_000
    left = {"device": torch.from_numpy(L).to(cuda), "numpy": L,
            "pinned": torch.from_numpy(L).pin_memory()}[left_kind]
    ms, _ = tensor_join_vectors(left, S, theta, device=cuda)      # S: pageable numpy
    assert np.array_equal(ms.lefts, ref[0]) and np.array_equal(ms.rights, ref[1])
    assert np.array_equal(ms.sims.view(np.uint32), ref[2].view(np.uint32))


def datagen_pair(nl, nr, dim, seed):
    from paper_2312_01476_b200 import datagen
    return datagen.clustered_pair(nl, nr, dim, 60, 0.4, seed)


# ---- raw-operand (bf16) wide path: BASELINE cfg4's bf16 relations ---------

def _bf16_tensor(x, dev):
    from paper_2312_01476_b200 import datagen
    return torch.from_numpy(datagen.bf16_bits(x).view(np.int16)).view(torch.bfloat16).to(dev)


def _bf16_case(nl, nr, dim, c, sigma, seed):
    from paper_2312_01476_b200 import datagen
    L, S = datagen.clustered_pair(nl, nr, dim, c, sigma, seed)
    L, S = datagen.round_bf16(L), datagen.round_bf16(S)
    L[5] = 0.0                              # a repaired row
    S[3, :] = 0.0
    S[3, 7] = np.float32(2.0 ** -100)       # below the repair threshold, not zero
    return L, S


@pytest.mark.parametrize("dim", [136, 200, 768])
def test_prepare_bf16(cuda, dim):
    """sjb_prepare_bf16: canonical fp32 rows bitwise the oracle's
    normalize_rows of the exact fp32 values, the raw bf16 operand image
    (component 0 := 1 for repaired rows), and RN(1 / ||x||)."""
    from paper_2312_01476_b200 import device as D
    L, _ = _bf16_case(700, 10, dim, 20, 0.6, dim)
    p = D.prepare_bf16(_bf16_tensor(L, cuda))
    want, rep = O.normalize_rows(L)
    assert np.array_equal(p.f32.cpu().numpy().view(np.uint32), want.view(np.uint32))
    assert p.repaired() == rep == 1
    rows, full = _decode_operand(p.op, len(L), dim)
    raw = L.copy()
    raw[5, 0] = 1.0                         # the reference's repaired row
    from paper_2312_01476_b200 import datagen
    assert np.array_equal(rows[:, :dim].view(np.uint16), datagen.bf16_bits(raw))
    assert (rows[:, dim:] == 0).all() and (full[len(L):] == 0).all()
    x64 = raw.astype(np.float64)
    ss = np.cumsum(x64 * x64, axis=1)[:, -1]            # sequential, exact squares
    inv = (1.0 / np.sqrt(ss)).astype(np.float32)
    got = p.inv_norm.cpu().numpy()
    assert np.array_equal(got[:len(L)].view(np.uint32), inv.view(np.uint32))
    assert (got[len(L):] == 0).all()


@pytest.mark.parametrize("theta", [0.75, 0.3, -1.0])
def test_bf16_join_exact_and_tensor_sims(cuda, theta):
    """The raw-operand filter (bf16 operands, normalise after the GEMM,
    band = sjb_raw_band): sims='exact' is bitwise the oracle's join of the
    fp32 values; sims='tensor' returns the same pair SET with every
    similarity within 1e-5 of the canonical one (the north star's bound)."""
    from paper_2312_01476_b200 import device as D
    from paper_2312_01476_b200.join import tensor_join_vectors
    nl, nr = (900, 2300) if theta > -1 else (300, 400)
    L, S = _bf16_case(nl, nr, 768, 30, 0.6, 17)
    wl, wr, ws = O.join_raw(L, S, theta, threads=4)
    assert len(wl) > 0
    pl, pr = D.prepare_bf16(_bf16_tensor(L, cuda)), D.prepare_bf16(_bf16_tensor(S, cuda))
    m = D.join_prepared(pl, pr, theta)
    lo, ro, so = m.to_host()
    assert np.array_equal(lo, wl) and np.array_equal(ro, wr)
    assert np.array_equal(so.view(np.uint32), ws.view(np.uint32))
    # raw band: far fewer non-matching candidates than the 16-bit per-row band
    mf = D.join_prepared(D.prepare(torch.from_numpy(L).to(cuda)),
                         D.prepare(torch.from_numpy(S).to(cuda)), theta)
    assert m.n_candidates <= mf.n_candidates
    for api in (False, True):
        if api:
            ms, _ = tensor_join_vectors(_bf16_tensor(L, cuda), _bf16_tensor(S, cuda), theta,
                                        sims="tensor")
            tl, tr, ts = ms.lefts, ms.rights, ms.sims
        else:
            tl, tr, ts = D.join_prepared(pl, pr, theta, sims="tensor").to_host()
        assert np.array_equal(tl, wl) and np.array_equal(tr, wr)
        err = np.abs(ts.astype(np.float64) - ws.astype(np.float64))
        assert err.max() <= 1e-5, err.max()
        assert (ts >= np.float32(theta)).all()


def test_bf16_overflow_retry_tensor_sims(cuda):
    """Tolerance emission under candidate overflow: the retry with the
    measured capacity returns the exact set."""
    from paper_2312_01476_b200 import device as D
    L, S = _bf16_case(600, 900, 256, 4, 0.4, 5)
    theta = 0.5
    wl, wr, ws = O.join_raw(L, S, theta, threads=4)
    pl, pr = D.prepare_bf16(_bf16_tensor(L, cuda)), D.prepare_bf16(_bf16_tensor(S, cuda))
    m = D.join_prepared(pl, pr, theta, cand_cap=4096, sims="tensor")
    assert m.retries >= 1
    lo, ro, so = m.to_host()
    assert np.array_equal(lo, wl) and np.array_equal(ro, wr)
    assert np.abs(so.astype(np.float64) - ws).max() <= 1e-5


@pytest.mark.parametrize("mma2", ["1", "2", "0"])
def test_wide_mma2_pair_kernel(cuda, monkeypatch, mma2):
    """Tensor sims on raw bf16 operands through the cta_group::2 wide kernel
    (default, SJB_WIDE_MMA2=2: 256 x 256 tiles per SM pair with two accumulator
    stages, operands by 2-SM tensor TMA; =1, -DSJB_AB_KERNELS=1 only: 256 x 512
    tiles, one accumulator tile -- the default library rejects that switch) and
    the 1-CTA kernel: odd R tile counts, partial pair tiles, an overflow
    retry -- the oracle's pair set, sims within 1e-5."""
    from paper_2312_01476_b200 import _lib, device as D
    if mma2 == "1" and not _lib.lib().sjb_ab_kernels():
        L, S = _bf16_case(300, 500, 384, 12, 0.5, 40)
        monkeypatch.setenv("SJB_WIDE_MMA2", mma2)
        with pytest.raises(_lib.SjbError, match="A/B kernel"):
            D.join_prepared(D.prepare_bf16(_bf16_tensor(L, cuda)),
                            D.prepare_bf16(_bf16_tensor(S, cuda)), 0.6, sims="tensor")
        return
    monkeypatch.setenv("SJB_WIDE_MMA2", mma2)
    for nl, nr, dim, seed in ((600, 1700, 384, 41), (1300, 2100, 256, 42), (200, 900, 768, 43),
                              (257, 513, 192, 44)):
        L, S = _bf16_case(nl, nr, dim, 12, 0.5, seed)
        theta = 0.6
        wl, wr, ws = O.join_raw(L, S, theta, threads=8)
        assert len(wl) > 0
        pl, pr = D.prepare_bf16(_bf16_tensor(L, cuda)), D.prepare_bf16(_bf16_tensor(S, cuda))
        for cap in (None, 4096):
            lo, ro, so = D.join_prepared(pl, pr, theta, sims="tensor", cand_cap=cap).to_host()
            assert np.array_equal(lo, wl) and np.array_equal(ro, wr), (nl, nr, dim, cap)
            assert np.abs(so.astype(np.float64) - ws).max() <= 1e-5


@pytest.mark.parametrize("grid", [0, 132, 131])
def test_bf16_tensor_sims_incremental_rounds(cuda, grid):
    """Tensor sims through the incremental join (JoinSession: the multi-GPU
    rounds' entry): S filtered in uneven row ranges that start on odd and even
    tiles, on the full grid, a reduced even grid (CTA pairs) and an odd grid
    (which falls back to the 1-CTA wide filter) -- the oracle's pair set, sims
    within 1e-5, identical to the one-launch join."""
    from paper_2312_01476_b200 import device as D
    L, S = _bf16_case(700, 2900, 384, 10, 0.6, 61)
    theta = 0.6
    wl, wr, ws = O.join_raw(L, S, theta, threads=8)
    assert len(wl) > 0
    pl, pr = D.prepare_bf16(_bf16_tensor(L, cuda)), D.prepare_bf16(_bf16_tensor(S, cuda))
    one = D.join_prepared(pl, pr, theta, sims="tensor").to_host()
    sess = D.JoinSession(pl, pr, theta, None, 0, grid=grid, sims="tensor")
    for r0, r1 in ((0, 256), (256, 1024), (1024, 1280), (1280, 2900)):
        sess.filter_rows(r0, r1)
    lo, ro, so = sess.finish().result().to_host()
    assert np.array_equal(lo, wl) and np.array_equal(ro, wr)
    assert np.abs(so.astype(np.float64) - ws).max() <= 1e-5
    assert np.array_equal(lo, one[0]) and np.array_equal(ro, one[1])
    if grid != 131:   # the same kernel and K order: the same accumulator bits
        assert np.array_equal(so.view(np.uint32), one[2].view(np.uint32))


@pytest.mark.parametrize("mode", ["rows", "group"])
def test_bf16_canonical_sims_row_grouped_recheck(cuda, monkeypatch, mode):
    """Canonical sims on raw bf16 operands: the default (1-CTA filter +
    tile-group recheck; any other value of SJB_WIDE_EXACT) and the A/B path
    SJB_WIDE_EXACT=rows (CTA-pair filter emitting candidates only and recording
    per-item segment offsets; items rechecked in the filter's order by warps
    that sort 2048 candidates by left row and stage each distinct left row
    once): the oracle's MatchSet bit for bit, one-launch and
    incremental, with an overflow retry, dims with a partial last chunk, rows
    with one candidate (warps spanning several left rows) and dense rows."""
    from paper_2312_01476_b200 import device as D
    monkeypatch.setenv("SJB_WIDE_EXACT", mode)
    cases = ((700, 2900, 384, 10, 0.6, 0.6, 71),      # clustered: dense rows
             (513, 1100, 260, 6, 0.7, 0.55, 72),      # dim % 32 != 0
             (300, 2300, 768, 300, 0.5, 0.7, 73),     # many small clusters: sparse rows
             (257, 513, 192, 4, 0.4, 0.5, 74))
    for nl, nr, dim, ncl, sigma, theta, seed in cases:
        L, S = _bf16_case(nl, nr, dim, ncl, sigma, seed)
        wl, wr, ws = O.join_raw(L, S, theta, threads=8)
        assert len(wl) > 0
        pl, pr = D.prepare_bf16(_bf16_tensor(L, cuda)), D.prepare_bf16(_bf16_tensor(S, cuda))
        for cap in (None, 4096):
            m = D.join_prepared(pl, pr, theta, cand_cap=cap)
            lo, ro, so = m.to_host()
            assert np.array_equal(lo, wl) and np.array_equal(ro, wr), (mode, dim, cap)
            assert np.array_equal(so.view(np.uint32), ws.view(np.uint32)), (mode, dim, cap)
        sess = D.JoinSession(pl, pr, theta, None, 0)
        step = 256 * max(1, (nr // 256) // 3)
        for r0 in range(0, nr, step):
            sess.filter_rows(r0, min(nr, r0 + step))
        lo, ro, so = sess.finish().result().to_host()
        assert np.array_equal(lo, wl) and np.array_equal(ro, wr)
        assert np.array_equal(so.view(np.uint32), ws.view(np.uint32))


def test_pending_recheck_staged_equals_gather(cuda, monkeypatch):
    """Tensor sims: the band pairs' canonical recheck with rows staged through
    shared memory by whole warps (default) against the thread-per-pair gather
    (SJB_PENDING=gather): the same MatchSet bit for bit (pending pairs carry
    the canonical chain's bits), and the oracle's pair set.  Dims that are not
    a multiple of the 32-element chunk end in a partial chunk."""
    from paper_2312_01476_b200 import device as D
    for nl, nr, dim, seed in ((700, 1900, 768, 51), (513, 1100, 260, 52), (300, 2300, 388, 53)):
        L, S = _bf16_case(nl, nr, dim, 6, 0.7, seed)
        theta = 0.55
        wl, wr, ws = O.join_raw(L, S, theta, threads=8)
        assert len(wl) > 0
        pl, pr = D.prepare_bf16(_bf16_tensor(L, cuda)), D.prepare_bf16(_bf16_tensor(S, cuda))
        out = {}
        for mode in ("staged", "gather"):
            monkeypatch.setenv("SJB_PENDING", mode)
            out[mode] = D.join_prepared(pl, pr, theta, sims="tensor").to_host()
            lo, ro, so = out[mode]
            assert np.array_equal(lo, wl) and np.array_equal(ro, wr), (dim, mode)
            assert np.abs(so.astype(np.float64) - ws).max() <= 1e-5
        assert np.array_equal(out["staged"][2].view(np.uint32), out["gather"][2].view(np.uint32))
        # some pairs were decided by the canonical chain: their sims are the oracle's bits
        assert (out["staged"][2].view(np.uint32) == ws.view(np.uint32)).any()


@pytest.mark.parametrize("pair", ["1", "0"])
def test_wide_pair_multicast(cuda, monkeypatch, pair):
    """A/B: wide-path tensor sims with CTA pairs sharing each S chunk by TMA
    multicast (SJB_WIDE_PAIR=1, built with -DSJB_AB_KERNELS=1; the default
    library rejects the switch); odd R block counts give the last pair a
    phantom block.  Same pair set as the oracle either way."""
    from paper_2312_01476_b200 import _lib, device as D
    if pair == "1" and not _lib.lib().sjb_ab_kernels():
        L, S = _bf16_case(300, 500, 384, 12, 0.5, 30)
        monkeypatch.setenv("SJB_WIDE_PAIR", pair)
        with pytest.raises(_lib.SjbError, match="A/B kernel"):
            D.join_prepared(D.prepare_bf16(_bf16_tensor(L, cuda)),
                            D.prepare_bf16(_bf16_tensor(S, cuda)), 0.6, sims="tensor")
        return
    monkeypatch.setenv("SJB_WIDE_PAIR", pair)
    for nl, nr, seed in ((600, 1700, 31), (1300, 2100, 32), (200, 900, 33)):
        L, S = _bf16_case(nl, nr, 384, 12, 0.5, seed)
        theta = 0.6
        wl, wr, ws = O.join_raw(L, S, theta, threads=8)
        assert len(wl) > 0
        pl, pr = D.prepare_bf16(_bf16_tensor(L, cuda)), D.prepare_bf16(_bf16_tensor(S, cuda))
        lo, ro, so = D.join_prepared(pl, pr, theta, sims="tensor").to_host()
        assert np.array_equal(lo, wl) and np.array_equal(ro, wr), (nl, nr)
        assert np.abs(so.astype(np.float64) - ws).max() <= 1e-5


def test_host_input_join_heavy_split(cuda, monkeypatch):
    """Output-heavy host-input joins split the left rows into 8 equal parts
    once the shape's previous result was large (join._result_bytes): the
    same canonical MatchSet, pinned and pageable inputs."""
    from paper_2312_01476_b200 import join as J
    L, S = O_pair(9000, 70_000, 16, 6, 0.5, 77)
    theta = 0.7
    wl, wr, ws = O.join_raw(L, S, theta, threads=8)
    assert len(wl) > 0
    monkeypatch.setattr(J, "HEAVY_RESULT_BYTES", 0)
    for pinned in (True, False):
        for _ in range(2):                        # the second call splits 8 ways
            lh = torch.from_numpy(L)
            sh = torch.from_numpy(S)
            if pinned:
                lh, sh = lh.pin_memory(), sh.pin_memory()
            ms, _ = J.tensor_join_vectors(lh, sh, theta, device=cuda)
            assert _bits_equal(ms, wl, wr, ws)
    assert max(J._result_bytes.values()) == len(wl) * 20


@pytest.mark.parametrize("sims", ["exact", "tensor"])
def test_bf16_vectors_api_in_parts(cuda, sims):
    """tensor_join_vectors on bf16 host tensors with >= 8 x 4096 left rows:
    the left rows join in 8 parts on the resident prepared S, each part's
    matches copied out while the next joins; the same set as the oracle."""
    from paper_2312_01476_b200.join import tensor_join_vectors
    L, S = _bf16_case(33_000, 2_500, 256, 40, 0.6, 23)
    theta = 0.8
    wl, wr, ws = O.join_raw(L, S, theta, threads=8)
    assert len(wl) > 0
    for pinned in (False, True):
        lt, st = _bf16_tensor(L, "cpu"), _bf16_tensor(S, "cpu")
        if pinned:
            lt, st = lt.pin_memory(), st.pin_memory()
        ms, stats = tensor_join_vectors(lt, st, theta, sims=sims, device=cuda)
        assert stats.pairs_compared == len(L) * len(S)
        assert np.array_equal(ms.lefts, wl) and np.array_equal(ms.rights, wr)
        if sims == "exact":
            assert np.array_equal(ms.sims.view(np.uint32), ws.view(np.uint32))
        else:
            assert np.abs(ms.sims.astype(np.float64) - ws).max() <= 1e-5


@pytest.mark.parametrize("world", [3, 8])
def test_owner_prepared_layout_on_device(cuda, manifest, golden, world):
    """The device side of multigpu.sharded_join_owned for `world` ranks on
    one GPU: every rank's pieces prepared into the padded buffers at their
    layout offsets (what the all-gathers deliver), then each rank's R shard
    filtered round by round (reduced grid but the last round) -- the shards
    concatenate to the golden cfg1 set, and the assembled prepared S equals
    a one-shot prepare (rows, operand image, errors, tile maxima)."""
    from paper_2312_01476_b200 import device as D
    from paper_2312_01476_b200 import multigpu as MG
    meta = manifest["cases"]["cfg1"]
    L, S = case_inputs(meta)
    lay = MG.piece_layout(len(S), world, rounds=3)
    assert lay.rounds == 3 and lay.rows >= len(S)
    Sd = torch.from_numpy(S).to(cuda)
    PR = D.empty_prepared(len(S), S.shape[1], cuda, rows=lay.rows)
    for k in range(world):
        local = torch.from_numpy(MG.local_pieces(S, lay, k)).to(cuda)
        off = 0
        for _, a, b in lay.owned(k):
            D.prepare_into(local[off:off + (b - a)], PR, a)
            off += b - a
    ref = D.prepare(Sd)
    n = len(S)
    assert torch.equal(PR.f32[:n], ref.f32)
    assert torch.equal(PR.op[:ref.op.numel()].view(torch.int16), ref.op.view(torch.int16))
    assert torch.equal(PR.row_err[:n], ref.row_err[:n])
    assert torch.equal(PR.tile_err[:D.tile_count(n)], ref.tile_err[:D.tile_count(n)])
    parts = []
    for k in range(world):
        r0, r1 = MG.shard_range(len(L), k, world)
        sess = D.JoinSession(D.prepare(torch.from_numpy(L[r0:r1]).to(cuda)), PR, meta["theta"],
                             None, r0)
        for j in range(lay.rounds):
            sess.filter_rows(*lay.round_rows(j), launch_grid=0 if j == lay.rounds - 1 else 100)
        parts.append(sess.finish().result().to_host())
    lo, ro, so = MG.concat_shards(parts)
    assert np.array_equal(lo, golden["cfg1_l"]) and np.array_equal(ro, golden["cfg1_r"])
    assert np.array_equal(so.view(np.uint32), golden["cfg1_s"].view(np.uint32))
