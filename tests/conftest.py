import json
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))

GOLDEN = os.path.join(HERE, "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libsjb200.so")


@pytest.fixture(scope="session")
def golden():
    return np.load(os.path.join(GOLDEN, "reference_outputs.npz"))


@pytest.fixture(scope="session")
def manifest():
    with open(os.path.join(GOLDEN, "manifest.json")) as fh:
        return json.load(fh)


def case_inputs(meta):
    """Regenerate the inputs of a golden join case (checked against its sha256)."""
    import hashlib
    from paper_2312_01476_b200 import datagen
    L, S = datagen.clustered_pair(meta["n_left"], meta["n_right"], meta["dim"],
                                  meta["centroids"], meta["sigma"], meta["seed"])
    if meta.get("zero_rows"):
        L[3] = 0
        S[7] = 0
    assert hashlib.sha256(L.tobytes()).hexdigest() == meta["sha_left"], "generator drift"
    assert hashlib.sha256(S.tobytes()).hexdigest() == meta["sha_right"], "generator drift"
    return L, S


def golden_tokens(golden):
    return bytes(golden["fnv_tokens"]).decode("utf-8").split("\x1f")


def rng():
    return np.random.default_rng(0x5EED)


@pytest.fixture
def small_relations():
    from paper_2312_01476_b200 import RawRelation
    return (RawRelation("left", [f"l_{i}" for i in range(40)]),
            RawRelation("right", [f"r_{i}" for i in range(30)]))


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2312_01476_b200 import build
    build.build()
    return torch.device("cuda", 0)
