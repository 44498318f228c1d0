"""Stress: many seeded shapes x sweep counts for the GS and Jacobi kernels
against the CPU oracle, bitwise (looks for rare races in the inter-CTA
protocols).  python tools/gs_stress.py [trials]"""
import hashlib
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "oracle"))
import torch  # noqa: E402

import oracle  # noqa: E402  (checker)
from paper_1004_1741_b200 import InitPattern, create_grid  # noqa: E402
from paper_1004_1741_b200.sweeps import execute  # noqa: E402

trials = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 2024)
bad = 0
for t in range(trials):
    ni = int(rng.integers(16, 400))  # odd ni: the pitched-copy paths
    nj, nk = (int(x) for x in rng.integers(4, 160, size=2))
    kernel = ("gs-naive", "gs-interleaved", "jacobi")[t % 3]
    iters = int(rng.integers(1, 12))
    depth = int(rng.integers(1, 5))
    host = create_grid(ni, nj, nk, InitPattern.seeded_random(t, -1.0, 1.0))
    want = oracle.run_serial(kernel, host.data, iters, 0.0, 1 / 6)
    dev = host.to_device("cuda:0")
    execute(kernel, dev, iters, 0.0, 1 / 6, depth)
    got = dev.data.cpu().numpy()
    ok = hashlib.sha256(got.tobytes()).digest() == hashlib.sha256(want.tobytes()).digest()
    bad += not ok
    print(f"{t:3d} {kernel:15s} {ni}x{nj}x{nk} iters={iters} depth={depth}: {'ok' if ok else 'MISMATCH'}",
          flush=True)
print(f"{trials - bad}/{trials} bitwise")
sys.exit(1 if bad else 0)
