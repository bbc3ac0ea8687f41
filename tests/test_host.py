"""Host-side logic that needs no GPU: API types, planner, C-ABI surface."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import REPO


def test_raw_relation_and_matchset():
    from paper_2312_01476_b200 import MatchSet, RawRelation, canonicalize
    r = RawRelation("R", ["a", "a"])
    assert len(r) == 2 and r.tokens == ("a", "a")
    m = MatchSet.from_rows("L", "R", [(1, 0, 0.9), (0, 0, 0.8), (0, 0, 0.8)])
    c = canonicalize(m)
    assert c.as_tuples() == [(0, 0, pytest.approx(0.8)), (1, 0, pytest.approx(0.9))]
    assert canonicalize(c) == c                       # idempotent
    assert MatchSet("L", "R") == canonicalize(MatchSet("L", "R"))
    with pytest.raises(ValueError):
        MatchSet("L", "R", np.zeros(1, np.uint64), np.zeros(2, np.uint64), np.zeros(1, np.float32))


def test_threshold_validation():
    from paper_2312_01476_b200 import Threshold
    assert Threshold.of(0.8).f32 == np.float32(0.8)
    for bad in (1.5, -1.01):
        with pytest.raises(ValueError):
            Threshold(bad)


def test_plan_batches(manifest):
    from paper_2312_01476_b200.join import plan_batches
    from paper_2312_01476_b200 import BudgetTooSmall
    p = plan_batches(1000, 1000, 100, 1_000_000)
    assert [p.left_block_rows, p.right_block_rows, len(p.tiles)] == manifest["plan_1000_1000_1MB"]
    with pytest.raises(BudgetTooSmall):
        plan_batches(10, 10, 4, 3)
    rng = np.random.default_rng(1)
    for _ in range(200):                               # exact cover
        nl, nr = int(rng.integers(0, 60)), int(rng.integers(0, 60))
        b = int(rng.integers(4, 20000))
        p = plan_batches(nl, nr, 8, b)
        cover = np.zeros((nl, nr), dtype=np.int32)
        for t in p.tiles:
            cover[t.left_row_start:t.left_row_start + t.left_row_count,
                  t.right_row_start:t.right_row_start + t.right_row_count] += 1
        assert (cover == 1).all()
        assert p.buffer_elems * 4 <= b or p.buffer_elems == 0 or b < 4


def test_host_embedding_twins(golden):
    """Single-token host twins of the model recipes match the reference bits."""
    from conftest import golden_tokens
    from paper_2312_01476_b200.embedding import fnv1a64, synthetic_vector
    toks = golden_tokens(golden)
    assert [fnv1a64(t.encode()) for t in toks] == golden["fnv_values"].tolist()
    want = golden["syn_16_7"]
    for i, t in enumerate(toks):
        v = synthetic_vector(fnv1a64(t.encode()) ^ 7, 16)
        assert np.array_equal(v.view(np.uint32), want[i].view(np.uint32))


def test_subword_host_twin_matches_oracle():
    import oracle as O
    from paper_2312_01476_b200.embedding import SubwordModel
    from paper_2312_01476_b200 import datagen
    table = datagen.bucket_table(997, 24, seed=3)
    toks = ["cat", "dogs", "abcdefghijkl", "xyz", "été"]
    m = SubwordModel(table)
    got = np.stack([m._vector(t) for t in toks])
    want = O.subword_embed(toks, table)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_datagen_deterministic():
    from paper_2312_01476_b200 import datagen
    a = datagen.clustered_pair(50, 40, 16, 5, 0.5, seed=9)
    b = datagen.clustered_pair(50, 40, 16, 5, 0.5, seed=9)
    assert all(np.array_equal(x, y) for x, y in zip(a, b))
    l1, r1 = datagen.strings(100, 120, seed=2)
    l2, r2 = datagen.strings(100, 120, seed=2)
    assert l1 == l2 and r1 == r2
    assert all(3 <= len(w) <= 12 for w in l1)


def _header_functions():
    src = open(os.path.join(REPO, "include", "simjoin_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sjb_[a-z0-9_]+)\s*\(", src)))


def test_c_abi_exports_every_declared_symbol():
    from paper_2312_01476_b200 import build
    path = build.build()
    lib = ctypes.CDLL(path)
    names = _header_functions()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), f"{n} declared in include/simjoin_b200.h but not exported"
    from paper_2312_01476_b200 import _lib
    assert set(names) <= set(_lib.EXPORTS)
    L = _lib.lib()
    assert L.sjb_version() == 1
    assert L.sjb_kpad(100) == 112 and L.sjb_kpad(4) == 16
    assert L.sjb_operand_elems(300, 100) == 512 * 112
    # 2e + e^2 + 4 d 2^-24 + 1e-6, e = u + 2^-25 sqrt(d): bf16 operands
    # (u = 2^-8) up to kpad 128, fp16 (u = 2^-11) above
    for d, u in ((100, 2.0 ** -8), (768, 2.0 ** -11)):
        e = u + 2.0 ** -25 * d ** 0.5
        want = 2 * e * (1 + 1e-6) + e * e + 4 * d * 2.0 ** -24 + 1e-6
        assert abs(L.sjb_default_band(d) - want) < 1e-9 * max(1.0, want * 1e3)
    assert 0.0078 < L.sjb_default_band(100) < 0.0079
    assert abs(L.sjb_accum_slack(100) - (4 * 100 * 2.0 ** -24 + 2e-6)) < 1e-9


def test_no_oracle_in_product():
    """The product package never imports or links the oracle."""
    pkg = os.path.join(REPO, "paper_2312_01476_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh")):
                txt = open(os.path.join(root, f)).read()
                assert "import oracle" not in txt and "refkern" not in txt, f
                assert "liboracle" not in txt and "from oracle" not in txt, f


def test_native_token_packer_matches_python():
    """csrc/sjb_pack.c (built by build()) packs exactly like the Python path:
    UTF-8 bytes back to back + NUL, int64 offsets; non-str tokens raise."""
    import numpy as np
    from paper_2312_01476_b200 import build as B, device as D
    B.build_pack()
    from paper_2312_01476_b200 import _sjbpack
    cases = [["l_0", "dog", "été", "", "a\0b", "x" * 300], [], [""], ["ascii"] * 1000]
    for toks in cases:
        data, offs = _sjbpack.pack(toks)
        enc = [t.encode("utf-8") for t in toks]
        assert data == b"".join(enc) + b"\0"
        want = np.concatenate([[0], np.cumsum([len(e) for e in enc], dtype=np.int64)])
        assert np.array_equal(np.frombuffer(offs, dtype=np.int64), want.astype(np.int64))
        b, o = D._pack_host(toks)
        assert bytes(b) == data and np.array_equal(o, want)
    with pytest.raises(TypeError):
        _sjbpack.pack(["a", 3])


def test_cost_model_matches_reference_goldens():
    """Estimates and plan choice equal the reference's cost model to the bit
    (tests/golden/cost_golden.json, made by running reference cost.py)."""
    import json
    import os
    from paper_2312_01476_b200.cost import CostParams, choose_plan, estimate_selection
    with open(os.path.join(os.path.dirname(__file__), "golden", "cost_golden.json")) as fh:
        cases = json.load(fh)["cases"]
    assert len(cases) > 50
    for c in cases:
        p = CostParams(**c["params"])
        plan, est = choose_plan(c["left"], c["right"], c["dim"], c["budget"], p)
        assert plan == c["plan"], c
        assert {k: float(v).hex() for k, v in est.items()} == c["estimates"], c
        assert float(estimate_selection(c["left"], c["dim"], p)).hex() == c["selection"]
    assert {c["plan"] for c in cases} >= {"tensor", "prefetch_nlj"}


def test_cost_params_validation_and_json():
    from paper_2312_01476_b200.cost import CostParams
    p = CostParams(1.0, 2.0, 3.0, 0.5, 0.25)
    assert CostParams.from_json(p.to_json()) == p and p.compare_ns(10) == 8.0
    for bad in (dict(access_ns=-1.0), dict(tensor_efficiency=0.0), dict(tensor_efficiency=1.5)):
        kw = dict(access_ns=1.0, model_ns=1.0, compare_base_ns=1.0, compare_per_dim_ns=1.0)
        kw.update(bad)
        with pytest.raises(ValueError):
            CostParams(**kw)
    with pytest.raises(ValueError, match="missing"):
        CostParams.from_dict({"access_ns": 1.0})


def test_bench_launcher_spawns_ranks():
    """bench.py --gpus 2 without a torchrun environment re-launches itself
    under torch.distributed.run with 2 ranks; rank 0 alone prints one JSON
    line whose n_gpus is the real world size.  (The reference arm needs no
    GPU, so the launcher is exercised here on CPU at cfg1.)"""
    import json
    import subprocess
    import sys
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference",
                          "--gpus", "2", "--config", "cfg1", "--steps", "1", "--warmup", "0",
                          "--nlj-pairs", "1e7"], capture_output=True, text=True, env=env,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 2 and rec["impl"] == "reference"
    assert rec["config"]["global_batch"] == 10_000 * 10_000
    assert rec["parity"]["matches"] == 52_884          # the golden cfg1 count
    assert rec["steps"] * rec["ms_per_step"] / 1e3 <= rec["cpu_baseline"]["full_wall_s"] * 2


def test_reference_package_matches_reference_kernels(manifest, golden):
    """The two CPU references agree: the unmodified package (baseline/_ref,
    simjoin.tensor_join) and its kernels built from source (oracle/_ref via
    refkern) give the golden cfg1 MatchSet bit for bit."""
    import simjoin_ref
    import refkern
    from conftest import case_inputs
    sj = simjoin_ref.load()
    if sj is None:
        pytest.skip(simjoin_ref.error())
    assert simjoin_ref.compiled(sj)
    meta = manifest["cases"]["cfg1"]
    L, S = case_inputs(meta)
    lt, rt = [f"l{i}" for i in range(len(L))], [f"r{i}" for i in range(len(S))]
    table = dict(zip(lt, L))
    table.update(zip(rt, S))
    ms, st = sj.tensor_join(sj.RawRelation("a", lt), sj.RawRelation("b", rt),
                            sj.LookupModel(table, L.shape[1]), meta["theta"], 64 << 20, threads=4)
    want = (golden["cfg1_l"], golden["cfg1_r"], golden["cfg1_s"])
    got = (np.asarray(ms.lefts), np.asarray(ms.rights), np.asarray(ms.sims))
    if refkern.available():
        lo, ro, so, _ = refkern.tensor_join_vectors(L, S, meta["theta"], threads=4)
        got2 = (lo, ro, so)
    else:
        got2 = got
    for g in (got, got2):
        assert np.array_equal(g[0], want[0]) and np.array_equal(g[1], want[1])
        assert np.array_equal(g[2].view(np.uint32), want[2].view(np.uint32))
