"""The ``cuda`` kernel backend inside the UNMODIFIED reference package.

The reference selects its kernels through ``simjoin.kernels`` (kernels.py:
18-60); a backend registered there is used by the reference's own operators
(join.py: tensor_join, nlj_prefetch, e_selection via linalg), by its
``backend`` test fixture (pkg/tests/conftest.py:23-29, parametrised over
``available_backends()``) and by its ``backends`` benchmark experiment
(bench.py:276-285).  These tests register paper_2312_01476_b200.kernels
there and run the reference's own code paths on it,
requiring results bitwise equal to the reference's compiled backend.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sj(cuda):
    import simjoin_ref
    mod = simjoin_ref.load()
    if mod is None:
        pytest.skip(simjoin_ref.error())
    assert simjoin_ref.compiled(mod)
    from paper_2312_01476_b200 import kernels as cuda_backend
    cuda_backend.register(mod.kernels)
    assert "cuda" in mod.kernels.available_backends()
    prev = mod.kernels.active_backend()
    yield mod
    mod.kernels.set_backend(prev)


def _cols(ms):
    return (np.asarray(ms.lefts, np.uint64), np.asarray(ms.rights, np.uint64),
            np.asarray(ms.sims, np.float32))


def _same(a, b):
    return (np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
            and np.array_equal(a[2].view(np.uint32), b[2].view(np.uint32)))


def _run_ops(sj, backend, left, right, model_fn, theta, budget):
    sj.kernels.set_backend(backend)
    out = {}
    m = model_fn()
    out["tensor"], st = sj.tensor_join(left, right, m, theta, budget, threads=2)
    out["tensor_stats"] = (st.pairs_compared, st.matches, st.model_calls_left,
                           st.model_calls_right)
    out["nlj"], _ = sj.nlj_prefetch(left, right, model_fn(), theta, threads=3)
    out["nlj_inner_left"], _ = sj.nlj_prefetch(left, right, model_fn(), theta, threads=2,
                                               inner="left")
    return out


@pytest.mark.parametrize("theta", [0.0, 0.3, -1.0])
def test_reference_fixture_shapes_on_cuda_backend(sj, theta):
    """The reference conftest's relations and model (small_relations,
    make_model: SyntheticModel(16, seed=7)) through the reference's own
    tensor_join and nlj_prefetch, cuda backend vs compiled backend."""
    left = sj.RawRelation("left", [f"l_{i}" for i in range(40)])
    right = sj.RawRelation("right", [f"r_{i}" for i in range(30)])
    mk = lambda: sj.SyntheticModel(16, seed=7)                     # noqa: E731
    want = _run_ops(sj, "compiled", left, right, mk, theta, 4096)
    got = _run_ops(sj, "cuda", left, right, mk, theta, 4096)
    for k in ("tensor", "nlj", "nlj_inner_left"):
        assert _same(_cols(got[k]), _cols(want[k])), k
    assert got["tensor_stats"] == want["tensor_stats"]


def test_reference_operators_clustered_on_cuda_backend(sj, manifest, golden):
    """A clustered cfg1-shaped join (LookupModel over the golden cfg1
    vectors) through the reference's operators on the cuda backend: the
    golden MatchSet the reference produced on its compiled backend."""
    from conftest import case_inputs
    meta = manifest["cases"]["cfg1"]
    L, S = case_inputs(meta)
    lt, rt = [f"l{i}" for i in range(len(L))], [f"r{i}" for i in range(len(S))]
    table = dict(zip(lt, L))
    table.update(zip(rt, S))
    model = sj.LookupModel(table, L.shape[1])
    sj.kernels.set_backend("cuda")
    want = (golden["cfg1_l"], golden["cfg1_r"], golden["cfg1_s"])
    ms, st = sj.tensor_join(sj.RawRelation("left", lt), sj.RawRelation("right", rt), model,
                            meta["theta"], 64 << 20, threads=4)
    assert _same(_cols(ms), want) and st.matches == meta["matches"]
    ms2, _ = sj.nlj_prefetch(sj.RawRelation("left", lt), sj.RawRelation("right", rt), model,
                             meta["theta"], threads=4)
    assert _same(_cols(ms2), want)


def test_reference_backends_experiment_includes_cuda(sj):
    """The reference's `backends` benchmark experiment (bench.py:276-285)
    iterates available_backends(): the registered cuda backend runs both
    algorithms and reports the compiled backend's match counts."""
    import importlib
    rows = importlib.import_module("simjoin.bench").run_experiment("backends", reps=1)
    by = {}
    for r in rows:
        by.setdefault(r["algo"], {})[r["experiment"]] = r["matches"]
    for algo, per in by.items():
        assert "backends[cuda]" in per and "backends[compiled]" in per, per
        assert per["backends[cuda]"] == per["backends[compiled]"], (algo, per)
        assert per["backends[cuda]"] > 0


def test_kernel_functions_bitwise(sj):
    """Every function of the backend contract (_ckern.pyx:41-212) on the
    cuda backend equals the compiled backend bit for bit."""
    K = sj.kernels
    cu, cc = K.get_backend("cuda"), K.get_backend("compiled")
    rng = np.random.default_rng(11)
    m = rng.standard_normal((300, 37), dtype=np.float32)
    m[4] = 0.0
    a, b = m.copy(), m.copy()
    assert cu.normalize_rows_inplace(a) == cc.normalize_rows_inplace(b)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    assert np.array_equal(cu.row_norms(m).view(np.uint32), cc.row_norms(m).view(np.uint32))
    assert np.array_equal(cu.dots_vm(a[0], a).view(np.uint32), cc.dots_vm(a[0], a).view(np.uint32))
    bt = cc.pack_transpose(a[:200])
    assert np.array_equal(cu.pack_transpose(a[:200]), bt)
    o1 = np.empty((100, 200), np.float32)
    o2 = np.empty((100, 200), np.float32)
    cu.tile_dot(a[100:200], bt, o1)
    cc.tile_dot(a[100:200], bt, o2)
    assert np.array_equal(o1.view(np.uint32), o2.view(np.uint32))
    h1, h2 = cu.scan_hits(o1, np.float32(0.1), 5, 7), cc.scan_hits(o2, np.float32(0.1), 5, 7)
    assert all(np.array_equal(x, y) for x, y in zip(h1, h2))
    c1 = cu.nlj_rows(a, 3, 250, a[:180], np.float32(0.2), np.float32(1e-4))
    c2 = cc.nlj_rows(a, 3, 250, a[:180], np.float32(0.2), np.float32(1e-4))
    cat = lambda ch: tuple(np.concatenate([c[k] for c in ch]) for k in range(3))  # noqa: E731
    g1, g2 = cat(c1), cat(c2)
    assert len(g2[0]) > 0
    assert np.array_equal(g1[0], g2[0]) and np.array_equal(g1[1], g2[1])
    assert np.array_equal(g1[2].view(np.uint32), g2[2].view(np.uint32))
    # rows that are NOT unit (the contract accepts any rows): raw dots >= theta
    big = a * np.float32(1.5)                 # norm 1.5 rows: dots up to 2.25
    c1 = cu.nlj_rows(big, 0, 300, big[:50], np.float32(0.6), np.float32(1e-4))
    c2 = cc.nlj_rows(big, 0, 300, big[:50], np.float32(0.6), np.float32(1e-4))
    g1, g2 = cat(c1), cat(c2)
    assert len(g2[0]) > 0
    assert np.array_equal(g1[0], g2[0]) and np.array_equal(g1[1], g2[1])
    assert np.array_equal(g1[2].view(np.uint32), g2[2].view(np.uint32))
    assert cu.fnv1a64(b"hello") == cc.fnv1a64(b"hello")
    s1, s2 = np.empty(16, np.float32), np.empty(16, np.float32)
    cu.synthetic_fill(12345, s1)
    cc.synthetic_fill(12345, s2)
    assert np.array_equal(s1.view(np.uint32), s2.view(np.uint32))
