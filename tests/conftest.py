import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libsb200.so")
    config.addinivalue_line("markers", "slow: long-running parity case")


def make_input(spec):
    """Rebuild a golden-fixture input grid (host numpy) from its spec."""
    from paper_1004_1741_b200.grid import InitPattern, create_grid, set_halo

    ni, nj, nk = spec["shape"]
    kind = spec["pattern"]
    if kind == "random":
        pat = InitPattern.seeded_random(spec["seed"], spec["lo"], spec["hi"])
    elif kind == "uniform":
        pat = InitPattern.uniform(spec["value"])
    else:
        pat = InitPattern.linear()
    g = create_grid(ni, nj, nk, pat)
    if spec.get("halo") is not None:
        set_halo(g, float(spec["halo"]))
    return g


def coeffs_of(rec):
    return tuple(float.fromhex(c) for c in rec["coeffs"])


def sha(a):
    import hashlib

    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


@pytest.fixture(scope="session")
def small_cases():
    meta = json.loads((GOLDEN / "small_cases.json").read_text())
    arrays = np.load(GOLDEN / "small_cases.npz")
    return {name: (rec, arrays[name]) for name, rec in meta.items()}


@pytest.fixture(scope="session")
def hashed_cases():
    return json.loads((GOLDEN / "hashes.json").read_text())
