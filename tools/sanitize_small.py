"""Small runs of every kernel family for compute-sanitizer (one tool per
run): fused single-grid Jacobi (depths 1-4, 8), GS (both associations),
the fused Jacobi slab exchange and the fused GS z-pipeline (3 slabs on one
GPU), each checked against the oracle."""
import ctypes
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "oracle"))
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_1004_1741_b200 import InitPattern, create_grid  # noqa: E402
from paper_1004_1741_b200.kernels import StencilCoeffs  # noqa: E402
from paper_1004_1741_b200.sweeps import SweepPlan, execute, run  # noqa: E402

ok = True
g = create_grid(70, 36, 30, InitPattern.seeded_random(3, -1.0, 1.0))
for kernel, depth in (("jacobi", 1), ("jacobi", 2), ("jacobi", 3), ("jacobi", 4), ("jacobi", 8),
                      ("gs-naive", 1), ("gs-interleaved", 1)):
    a = 0.25 if kernel == "jacobi" else 0.0
    want = oracle.run_serial(kernel, g.data, 9, a, 1 / 6)
    d = g.to_device("cuda:0")
    execute(kernel, d, 9, a, 1 / 6, depth)
    same = np.array_equal(d.data.cpu().numpy(), want)
    ok &= same
    print(kernel, depth, "ok" if same else "MISMATCH", flush=True)
for kernel in ("jacobi", "gs-naive"):
    a = 0.25 if kernel == "jacobi" else 0.0
    h = create_grid(70, 36, 30, InitPattern.seeded_random(4, -1.0, 1.0))
    want = oracle.run_serial(kernel, h.data, 7, a, 1 / 6)
    variant = "threaded" if kernel == "jacobi" else "pipeline"
    out = run(SweepPlan(kernel, variant, 7, coeffs=StencilCoeffs(a, 1 / 6)), h, devices=[0, 0, 0])
    same = np.array_equal(out.data, want)
    ok &= same
    print(kernel, "3 slabs", "ok" if same else "MISMATCH", flush=True)
sys.exit(0 if ok else 1)
