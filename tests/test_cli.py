"""The `simjoin join` surface (paper_2312_01476_b200.cli) against the
reference CLI (cli.py:40-300): model-spec grammar, vec-file parsing, token
files and exit codes on CPU; on the GPU, the matches file must be
byte-identical and the RunRecord equal field by field (except the run's
wall time, timestamp and peak_buffer_bytes -- no dense buffer exists here)
to the reference CLI's for the same inputs."""
import json
import os

import numpy as np
import pytest

from paper_2312_01476_b200 import cli


def test_model_spec_grammar():
    s = cli.ModelSpec("synthetic:seed=7:dim=16")
    assert (s.kind, s.seed, s.dim, s.latency_ns) == ("synthetic", 7, 16, 0)
    s = cli.ModelSpec("synthetic:seed=1:dim=4:latency_ns=9")
    assert s.latency_ns == 9
    v = cli.ModelSpec("vec:/a/b:c.vec:oov=synthetic")
    assert (v.kind, v.path, v.oov) == ("vec", "/a/b:c.vec", "synthetic")
    assert cli.ModelSpec("vec:x.vec").oov == "error"
    for bad in ("synthetic:seed=1", "synthetic:seed=x:dim=3", "synthetic:seed=1:dim=2:foo=3",
                "vec:", "vec:p:oov=maybe", "glove:x"):
        with pytest.raises(ValueError):
            cli.ModelSpec(bad)


def test_vec_file_parsing(tmp_path):
    from paper_2312_01476_b200.errors import ParseError
    p = tmp_path / "m.vec"
    p.write_text("3 2\na 1 0\nb 0.5 0.25\na 2 2\n")
    m = cli.load_vec_file(str(p))
    assert m.dim == 2 and len(m) == 2
    assert np.array_equal(m.embed("a"), np.array([2, 2], np.float32))     # last duplicate wins
    cases = {"": 1, "3\n": 1, "x 2\n": 1, "-1 2\n": 1, "2 2\na 1 0\n": 3, "1 2\na 1\n": 2,
             "1 2\na 1 x\n": 2, "1 2\na 1 inf\n": 2, "1 2\na 1 0\nextra\n": 3}
    for text, line in cases.items():
        p.write_text(text)
        with pytest.raises(ParseError) as ei:
            cli.load_vec_file(str(p))
        assert ei.value.line == line, text


def test_gen_relation_and_exit_codes(tmp_path, capsys):
    out = tmp_path / "t.txt"
    assert cli.main(["gen", "--rows", "5", "--seed", "3", "--out", str(out)]) == 0
    assert out.read_text() == "".join(f"tok_3_{i}\n" for i in range(5))
    r = cli.read_relation(str(out), "x")
    assert r.tokens == tuple(f"tok_3_{i}" for i in range(5))
    assert cli.main(["gen", "--rows", "-1", "--out", str(out)]) == cli.EXIT_USAGE
    args = ["join", str(out), str(out), "--model", "synthetic:seed=1:dim=4", "--out-matches",
            str(tmp_path / "m"), "--out-stats", str(tmp_path / "s")]
    assert cli.main(args + ["--theta", "1.5"]) == cli.EXIT_USAGE
    assert cli.main(args + ["--theta", "0.5", "--algo", "naive"]) == cli.EXIT_USAGE
    bad = args.copy()
    bad[4] = "vec:" + str(tmp_path / "missing.vec")
    assert cli.main(bad + ["--theta", "0.5"]) == cli.EXIT_IO
    with pytest.raises(SystemExit) as ei:
        cli.main(["join", "--theta", "0.5"])
    assert ei.value.code == cli.EXIT_USAGE
    err = capsys.readouterr().err
    assert all(ln.startswith("error: ") for ln in err.strip().splitlines())


def _reference_cli(argv):
    import simjoin_ref
    sj = simjoin_ref.load()
    if sj is None:
        pytest.skip(simjoin_ref.error())
    import importlib
    return importlib.import_module("simjoin.cli").main(argv)


def _write_vec(path, tokens, rows):
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(f"{len(tokens)} {rows.shape[1]}\n")
        for t, r in zip(tokens, rows):
            fh.write(t + " " + " ".join(np.format_float_positional(x, unique=True, trim="-")
                                        for x in r) + "\n")


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["cfg1_vec_tensor", "cfg1_vec_prefetch", "synthetic"])
def test_cli_join_matches_reference(cuda, manifest, tmp_path, case):
    """cfg1 (the reference's CPU-sized config) through both CLIs."""
    from conftest import case_inputs
    if case == "synthetic":
        lt = [f"l_{i}" for i in range(3000)]
        rt = [f"r_{i}" for i in range(2000)]
        model, theta, algo = "synthetic:seed=7:dim=100", "0.3", "tensor"
    else:
        meta = manifest["cases"]["cfg1"]
        L, S = case_inputs(meta)
        lt = [f"L{i}" for i in range(len(L))]
        rt = [f"S{i}" for i in range(len(S))]
        _write_vec(tmp_path / "m.vec", lt + rt, np.concatenate([L, S]))
        model, theta = f"vec:{tmp_path / 'm.vec'}", str(meta["theta"])
        algo = case.rsplit("_", 1)[1]
    (tmp_path / "l.txt").write_text("".join(t + "\n" for t in lt))
    (tmp_path / "r.txt").write_text("".join(t + "\n" for t in rt))
    outs = {}
    for who, fn in (("ours", cli.main), ("ref", _reference_cli)):
        m, s = tmp_path / f"{who}.csv", tmp_path / f"{who}.json"
        rc = fn(["join", str(tmp_path / "l.txt"), str(tmp_path / "r.txt"), "--model", model,
                 "--theta", theta, "--algo", algo, "--threads", "4", "--out-matches", str(m),
                 "--out-stats", str(s)])
        assert rc == 0, who
        outs[who] = (m.read_bytes(), json.loads(s.read_text()), list(json.loads(s.read_text())))
    assert outs["ours"][0] == outs["ref"][0] and len(outs["ref"][0]) > 0
    assert outs["ours"][2] == outs["ref"][2]                         # same fields, same order
    skip = {"wall_nanos", "timestamp", "peak_buffer_bytes"}
    for k in outs["ref"][1]:
        if k not in skip:
            assert outs["ours"][1][k] == outs["ref"][1][k], k
