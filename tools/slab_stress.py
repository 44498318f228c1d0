"""Stress the fused slab exchanges: many seeded shapes x slab counts x sweep
counts through run(threaded / pipeline plan, devices=[0] * G) -- the fused
Jacobi edge-plane stores (depths 1-8) and the fused GS z-pipeline (ghost
pushes, per-(sweep, J) flags) -- bitwise against the CPU oracle.

    python tools/slab_stress.py [trials] [seed]
"""
import hashlib
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "oracle"))
import torch  # noqa: E402,F401

import oracle  # noqa: E402  (checker)
from paper_1004_1741_b200 import InitPattern, create_grid  # noqa: E402
from paper_1004_1741_b200.kernels import StencilCoeffs  # noqa: E402
from paper_1004_1741_b200.sweeps import SweepPlan, run  # noqa: E402
from paper_1004_1741_b200.sweeps import engine  # noqa: E402

trials = int(sys.argv[1]) if len(sys.argv) > 1 else 60
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 7)
bad = 0
for t in range(trials):
    kernel = ("gs-naive", "gs-interleaved", "jacobi")[t % 3]
    ni = int(rng.integers(8, 300)) * (2 if t % 5 else 1)  # mostly even ni (the fused paths)
    nj = int(rng.integers(2, 120))
    G = int(rng.integers(2, 10))
    nk = int(rng.integers(G, 140))
    iters = int(rng.integers(1, 15))
    depth = int(rng.integers(1, 9))
    a, b = (0.3, 0.11) if kernel == "jacobi" else (0.0, 1 / 6)
    host = create_grid(ni, nj, nk, InitPattern.seeded_random(1000 + t, -1.0, 1.0))
    want = oracle.run_serial(kernel, host.data, iters, a, b)
    engine.DEFAULT_DEPTH = depth
    variant = "threaded" if kernel == "jacobi" else "pipeline"
    out = run(SweepPlan(kernel, variant, iters, coeffs=StencilCoeffs(a, b)), host, devices=[0] * G)
    ok = hashlib.sha256(out.data.tobytes()).digest() == hashlib.sha256(want.tobytes()).digest()
    bad += not ok
    print(f"{t:3d} {kernel:15s} {ni}x{nj}x{nk} slabs={G} iters={iters} depth={depth}: "
          f"{'ok' if ok else 'MISMATCH'}", flush=True)
print(f"{trials - bad}/{trials} bitwise")
sys.exit(1 if bad else 0)
