"""Golden records of the reference's WAVEFRONT engines (their schedule, not
just their result): run in the build container, where /root/reference
exists.

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_wavefront_golden.py

Writes ``wavefront_cases.json``: for each (kernel, grid, sweeps, groups N,
threads per group t, blocks B) the reference's run_wavefront
(pkg/src/stencilbench/sweeps/wavefront.py:127-376) output sha256 and its
stats["barrier_phases"] / stats["line_updates"].  tests/test_oracle.py pins
the C port of those engines (oracle/sb_oracle.c, the CPU baseline's
"wavefront" leg) to these records.
"""

import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))

from make_golden import GC, JC, make_input, sha, spec  # noqa: E402  (imports the reference)
from stencilbench.kernels import StencilCoeffs  # noqa: E402
from stencilbench.sweeps import SweepPlan, WavefrontConfig, run  # noqa: E402

CASES = [
    # kernel, shape, iters, coeffs, N, t, B
    ("jacobi", (18, 18, 18), 8, JC, 1, 2, 1),
    ("jacobi", (18, 18, 18), 8, JC, 1, 4, 3),
    ("jacobi", (18, 18, 18), 8, JC, 2, 2, 4),
    ("jacobi", (18, 18, 18), 8, JC, 2, 4, 5),
    ("jacobi", (17, 13, 11), 6, GC, 3, 2, 6),
    ("jacobi", (20, 9, 7), 4, JC, 1, 1, 1),
    ("jacobi", (20, 9, 7), 3, JC, 2, 1, 4),
    ("jacobi", (12, 16, 10), 8, JC, 2, 8, 2),
    ("jacobi", (9, 5, 12), 4, JC, 1, 4, 5),     # width-1 blocks
    ("gs-naive", (18, 18, 18), 8, GC, 1, 4, 2),
    ("gs-naive", (18, 18, 18), 6, GC, 2, 3, 5),
    ("gs-interleaved", (18, 18, 18), 6, GC, 2, 2, 3),
    ("gs-interleaved", (15, 11, 9), 5, GC, 3, 1, 4),
    ("gs-naive", (9, 5, 12), 4, GC, 2, 4, 5),
]


def main():
    out = []
    for kernel, shape, iters, coeffs, n, t, B in CASES:
        sp = spec(shape, lo=-1.0 if kernel != "jacobi" else 0.0)
        g = make_input(sp)
        in_hash = sha(g.data)
        plan = SweepPlan(kernel, "wavefront", iters, coeffs=StencilCoeffs(*coeffs),
                         config=WavefrontConfig(num_groups=n, threads_per_group=t, blocks=B))
        stats = {}
        res = run(plan, g, stats=stats)
        out.append({"kernel": kernel, "spec": sp, "iters": iters,
                    "coeffs": [float(c).hex() for c in coeffs], "groups": n, "tpg": t, "blocks": B,
                    "input_sha256": in_hash, "output_sha256": sha(res.data),
                    "barrier_phases": int(stats["barrier_phases"]),
                    "line_updates": int(stats["line_updates"])})
        print(kernel, shape, iters, n, t, B, stats["barrier_phases"], flush=True)
    (HERE / "wavefront_cases.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
