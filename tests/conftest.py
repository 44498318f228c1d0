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
    """sha256 of the C-order little-endian float64 bytes (hashed plane by
    plane: no copy of a multi-GB grid)."""
    import hashlib

    a = np.ascontiguousarray(a, dtype="<f8")
    h = hashlib.sha256()
    for plane in a.reshape(a.shape[0], -1) if a.ndim > 1 else [a]:
        h.update(memoryview(plane))
    return h.hexdigest()


def sha_device(t, chunk_planes=64):
    """sha() of a CUDA float64 tensor, downloaded a few planes at a time."""
    import hashlib

    import torch

    h = hashlib.sha256()
    buf = None
    for k0 in range(0, t.shape[0], chunk_planes):
        part = t[k0:k0 + chunk_planes]
        if buf is None or buf.shape != part.shape:
            buf = torch.empty(part.shape, dtype=t.dtype, pin_memory=True)
        buf.copy_(part)
        a = buf.numpy()
        for plane in a.reshape(a.shape[0], -1):
            h.update(memoryview(plane))
    return h.hexdigest()


@pytest.fixture(scope="session")
def small_cases():
    meta = json.loads((GOLDEN / "small_cases.json").read_text())
    arrays = np.load(GOLDEN / "small_cases.npz")
    return {name: (rec, arrays[name]) for name, rec in meta.items()}


@pytest.fixture(scope="session")
def hashed_cases():
    return json.loads((GOLDEN / "hashes.json").read_text())
