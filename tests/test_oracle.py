"""The CPU oracle (oracle/sj_oracle.c) against the reference's own outputs.

Pins the oracle: tests/golden/reference_outputs.npz was produced by running
the reference package (compiled backend) -- see tests/golden/make_golden.py.
"""
import numpy as np
import pytest

import oracle as O
from conftest import case_inputs, golden_tokens

JOIN_CASES = ["c_small", "c_d4", "c_d64", "c_d16_neg", "c_one", "c_ragged", "c_all", "cfg1",
              "c_d200", "c_d768"]


def test_normalize_kat(golden):
    out, rep = O.normalize_rows(golden["kat_norm_in"])
    assert np.array_equal(out.view(np.uint32), golden["kat_norm_out"].view(np.uint32))
    assert rep == int(golden["kat_norm_repaired"][0]) == 2
    assert np.allclose(out[0], [0.6, 0.8])
    assert np.array_equal(out[1], [1.0, 0.0])       # SPEC.md:219 repair rule


def test_fnv(golden):
    toks = golden_tokens(golden)
    got = O.fnv1a64_many(toks)
    assert np.array_equal(got, golden["fnv_values"])


@pytest.mark.parametrize("dim,seed", [(16, 7), (4, 1), (100, 0)])
def test_synthetic_model(golden, dim, seed):
    toks = golden_tokens(golden)
    seeds = O.fnv1a64_many(toks, seed)
    got = O.synthetic_fill_many(seeds, dim)
    assert np.array_equal(got.view(np.uint32), golden[f"syn_{dim}_{seed}"].view(np.uint32))


def test_nlj_kat(golden):
    s2 = np.float32(1 / np.sqrt(2))
    L = np.array([[1, 0], [0, 1]], dtype=np.float32)
    S = np.array([[1, 0], [s2, s2]], dtype=np.float32)
    lo, ro, so = O.join_raw(L, S, 0.5)
    assert list(zip(lo.tolist(), ro.tolist())) == [(0, 0), (0, 1), (1, 1)]
    assert np.array_equal(lo, golden["kat_nlj_l"]) and np.array_equal(ro, golden["kat_nlj_r"])
    assert np.array_equal(so.view(np.uint32), golden["kat_nlj_s"].view(np.uint32))


@pytest.mark.parametrize("theta", [0.0, 0.3, -1.0])
def test_synthetic_join(golden, theta):
    toks_l = [f"l_{i}" for i in range(40)]
    toks_r = [f"r_{i}" for i in range(30)]
    L = O.synthetic_fill_many(O.fnv1a64_many(toks_l, 7), 16)
    S = O.synthetic_fill_many(O.fnv1a64_many(toks_r, 7), 16)
    lo, ro, so = O.join_raw(L, S, theta)
    k = f"synjoin_{theta}"
    assert np.array_equal(lo, golden[k + "_l"]) and np.array_equal(ro, golden[k + "_r"])
    assert np.array_equal(so.view(np.uint32), golden[k + "_s"].view(np.uint32))


@pytest.mark.parametrize("name", JOIN_CASES)
def test_clustered_join(golden, manifest, name):
    meta = manifest["cases"][name]
    L, S = case_inputs(meta)
    lo, ro, so = O.join_raw(L, S, meta["theta"], threads=8)
    assert len(lo) == meta["matches"]
    assert np.array_equal(lo, golden[name + "_l"])
    assert np.array_equal(ro, golden[name + "_r"])
    assert np.array_equal(so.view(np.uint32), golden[name + "_s"].view(np.uint32))


def test_reference_kernels_agree_with_oracle(golden, manifest):
    """oracle/_ref (the reference's own C, built by oracle/Makefile) driven by
    the restated orchestration reproduces the golden cfg1 result too."""
    import refkern
    if not refkern.available():
        pytest.skip("oracle/_ref not built (run `make -C oracle ref` where /root/reference exists)")
    meta = manifest["cases"]["c_ragged"]
    L, S = case_inputs(meta)
    lo, ro, so, st = refkern.tensor_join_vectors(L, S, meta["theta"], budget_bytes=1 << 16,
                                                 threads=4)
    assert np.array_equal(lo, golden["c_ragged_l"]) and np.array_equal(ro, golden["c_ragged_r"])
    assert np.array_equal(so.view(np.uint32), golden["c_ragged_s"].view(np.uint32))
    # the resumable row kernel (nlj_rows) agrees as well
    nl, _ = refkern.normalize_rows(L)
    nr, _ = refkern.normalize_rows(S)
    chunks = refkern.nlj_rows(nl, 0, nl.shape[0], nr, meta["theta"])
    cl = np.concatenate([c[0] for c in chunks])
    assert np.array_equal(cl, lo)


def test_cosine_vm_restatement_matches_reference(golden):
    """cosine_vm (linalg.py:70-84) restated on the oracle kernels: fp32
    na * norm_i, then fp32 dot / denom -- bitwise the reference's output."""
    a, m = golden["cos_vm_a"], golden["cos_vm_m"]
    na = O.row_norms(a.reshape(1, -1))[0]
    denom = np.multiply(np.float32(na), O.row_norms(m), dtype=np.float32)
    got = np.divide(O.dots_vm(a, m), denom, dtype=np.float32)
    assert np.array_equal(got.view(np.uint32), golden["cos_vm_out"].view(np.uint32))


def test_matches_file_format_restatement_pinned_to_numpy():
    """The Dragon4 restatement (oracle/fmt_oracle.py) equals numpy's
    format_float_positional(unique=True, trim='-') -- the reference's _fmt_sim
    (cli.py:99-102) -- on sweeps, powers of two, denormals and random bits."""
    import fmt_oracle as F
    bits = F.probe_bits(20000)
    vals = bits.view(np.float32)
    bad = [hex(int(b)) for b, v in zip(bits, vals) if F.fmt_sim(v) != F.fmt_sim_numpy(v)]
    assert not bad, bad[:5]
    for v, want in ((0.0, "0"), (-0.0, "-0"), (1.0, "1"), (0.5, "0.5"), (100.0, "100"),
                    (np.inf, "inf"), (-np.inf, "-inf"), (np.nan, "nan"), (0.1, "0.1"),
                    (np.float32(0.8), "0.8"), (1e-45, "0." + "0" * 44 + "1")):
        assert F.fmt_sim(v) == F.fmt_sim_numpy(v) == want, v
    assert (F.matches_file_reference([0, 2**64 - 1], [5, 7], np.float32([0.25, -1.0]))
            == b"0,5,0.25\n18446744073709551615,7,-1\n")
