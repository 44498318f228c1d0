"""Generate the golden fixtures by running the REFERENCE package itself.

Run in the build container (the only place /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py [--big]

Outputs (committed; nothing at test time reads /root/reference):

* ``small_cases.npz`` -- full padded result arrays of small sweeps computed
  by the reference's ``run_serial`` (pkg/src/stencilbench/sweeps/serial.py:8)
  with the reference's numba kernels (kernels.py:125-187), plus the
  independent scalar oracle of the reference tests (pkg/tests/reference.py)
  as a cross-check at generation time.
* ``hashes.json`` -- sha256 of the full padded result array (C order,
  little-endian float64) for the BASELINE.json configs and their prefixes,
  with a few sampled values for diagnostics.  ``--big`` adds the 512^3 x 100
  configs 3 and 5 (minutes of CPU).

Inputs are never stored: they are regenerated bit-identically from
numpy's PCG64 ``default_rng(seed)`` (reference grid.py:115-121) by
``paper_1004_1741_b200.grid.create_grid``; each record carries the sha256
of the input so a generator drift is caught, not silently absorbed.
"""

import argparse
import hashlib
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
HERE = Path(__file__).resolve().parent

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, REF_SRC)
sys.path.insert(0, REF_TESTS)

from stencilbench.grid import InitPattern, create_grid  # noqa: E402
from stencilbench.kernels import HAVE_NUMBA, StencilCoeffs  # noqa: E402
from stencilbench.sweeps import SweepPlan, run, run_serial  # noqa: E402
import reference as scalar_ref  # noqa: E402  (pkg/tests/reference.py)

JC = (0.5, 0.1)            # reference tests' Jacobi coefficients
GC = (0.0, 1.0 / 6.0)      # reference default / GS coefficients


def sha(a):
    """sha256 of the C-order little-endian float64 bytes, hashed plane by
    plane so a 17 GB grid is never duplicated in host memory."""
    a = np.ascontiguousarray(a, dtype="<f8")
    h = hashlib.sha256()
    for plane in a.reshape(a.shape[0], -1):
        h.update(memoryview(plane))
    return h.hexdigest()


def make_input(spec):
    ni, nj, nk = spec["shape"]
    kind = spec["pattern"]
    if kind == "random":
        g = create_grid(ni, nj, nk, InitPattern.seeded_random(spec["seed"], spec["lo"], spec["hi"]))
    elif kind == "uniform":
        g = create_grid(ni, nj, nk, InitPattern.uniform(spec["value"]))
    elif kind == "linear":
        g = create_grid(ni, nj, nk, InitPattern.linear())
    else:
        raise ValueError(kind)
    if spec.get("halo") is not None:  # BASELINE config 3: Dirichlet halo 1.0
        h = float(spec["halo"])
        d = g.data
        d[0], d[-1] = h, h
        d[:, 0], d[:, -1] = h, h
        d[:, :, 0], d[:, :, -1] = h, h
    return g


def spec(shape, pattern="random", seed=42, lo=0.0, hi=1.0, value=0.0, halo=None):
    return {"shape": list(shape), "pattern": pattern, "seed": seed, "lo": lo,
            "hi": hi, "value": value, "halo": halo}


def ref_result(kernel, sp, iters, coeffs, variant="serial", **kw):
    g = make_input(sp)
    in_hash = sha(g.data)
    plan = SweepPlan(kernel, variant, iters, coeffs=StencilCoeffs(*coeffs), **kw)
    out = run_serial(plan, g) if variant == "serial" else run(plan, g)
    # the engines return a grid the caller owns (g or the scratch copy)
    return in_hash, out.data


SMALL = [
    # name, kernel, spec, iters, coeffs        (reference test it mirrors)
    ("serial8_jacobi", "jacobi", spec((8, 8, 8)), 3, JC),            # test_sweeps_serial.py:26-32
    ("serial8_gsn", "gs-naive", spec((8, 8, 8)), 3, GC),
    ("serial8_gsi", "gs-interleaved", spec((8, 8, 8)), 3, GC),
    ("ident6_jacobi", "jacobi", spec((6, 6, 6)), 7, (1.0, 0.0)),      # :19-23
    ("halo678_jacobi", "jacobi", spec((6, 7, 8)), 2, GC),             # :35-42
    ("halo678_gsn", "gs-naive", spec((6, 7, 8)), 2, GC),
    ("halo678_gsi", "gs-interleaved", spec((6, 7, 8)), 2, GC),
    ("det765_jacobi", "jacobi", spec((7, 6, 5)), 5, (0.2, 0.13)),     # :56-63
    ("wf18_jacobi", "jacobi", spec((18, 18, 18)), 8, JC),             # test_wavefront.py:46-57
    ("wf18_gsn", "gs-naive", spec((18, 18, 18)), 8, GC),
    ("wf18_gsi", "gs-interleaved", spec((18, 18, 18)), 6, GC),
    ("nc7135_jacobi", "jacobi", spec((7, 13, 5)), 4, JC),             # :60-63
    ("nc5921_jacobi", "jacobi", spec((5, 9, 21)), 4, JC),
    ("nc7135_gsn", "gs-naive", spec((7, 13, 5)), 4, GC),
    ("nc5921_gsn", "gs-naive", spec((5, 9, 21)), 4, GC),
    ("slim4126_jacobi", "jacobi", spec((4, 12, 6)), 4, JC),           # :66-70
    ("slim4126_gsn", "gs-naive", spec((4, 12, 6)), 4, GC),
    ("shallow441_jacobi", "jacobi", spec((4, 4, 1)), 2, JC),          # :157-163
    ("shallow441_gsn", "gs-naive", spec((4, 4, 1)), 2, GC),
    ("shallow482_gsi", "gs-interleaved", spec((4, 8, 2)), 4, GC),
    ("line1_gsi", "gs-interleaved", spec((1, 5, 4)), 3, GC),          # ni<2 fallback kernels.py:168
    ("line2_gsi", "gs-interleaved", spec((2, 3, 3)), 3, GC),
    ("thr34_jacobi", "jacobi", spec((34, 34, 34)), 8, JC),            # test_sweeps_threaded.py:31-36
    ("thr34_gsn", "gs-naive", spec((34, 34, 34)), 4, GC),
    ("thr34_gsi", "gs-interleaved", spec((34, 34, 34)), 4, GC),
    ("mixed16_gsn", "gs-naive", spec((16, 16, 16), lo=-1.0, hi=1.0), 5, GC),   # config-5 data
    ("mixed16_gsi", "gs-interleaved", spec((16, 16, 16), lo=-1.0, hi=1.0), 5, GC),
    ("halo1_24_jacobi", "jacobi", spec((24, 20, 22), halo=1.0), 9, GC),        # config-3 data
    ("uniform16_jacobi", "jacobi", spec((16, 16, 16), "uniform", value=3.0), 4, GC),  # test_acceptance.py:92-104
    ("uniform16_gsn", "gs-naive", spec((16, 16, 16), "uniform", value=3.0), 4, GC),
    ("uniform16_gsi", "gs-interleaved", spec((16, 16, 16), "uniform", value=3.0), 4, GC),
    ("linear16_jacobi", "jacobi", spec((16, 16, 16), "linear"), 4, GC),
    ("linear16_gsn", "gs-naive", spec((16, 16, 16), "linear"), 4, GC),
    ("linear16_gsi", "gs-interleaved", spec((16, 16, 16), "linear"), 4, GC),
    ("odd33_jacobi", "jacobi", spec((33, 31, 29)), 7, JC),
    ("even40_jacobi_a0", "jacobi", spec((40, 36, 30)), 11, GC),
    ("even40_gsn", "gs-naive", spec((40, 36, 30)), 3, GC),
    ("zero_iters_jacobi", "jacobi", spec((5, 5, 5)), 0, GC),
]

# (name, kernel, spec, iters list, coeffs)
HASHED = [
    ("cfg1_jacobi128", "jacobi", spec((128, 128, 128)), [1, 2, 20], GC),
    ("cfg2_gsn128", "gs-naive", spec((128, 128, 128)), [1, 20], GC),
    ("cfg2_gsi128", "gs-interleaved", spec((128, 128, 128)), [1, 20], GC),
    ("jacobi128_jc", "jacobi", spec((128, 128, 128)), [5], JC),
    ("mixed64_gsn", "gs-naive", spec((64, 64, 64), lo=-1.0, hi=1.0), [20], GC),
    ("mixed64_gsi", "gs-interleaved", spec((64, 64, 64), lo=-1.0, hi=1.0), [20], GC),
    ("cfg3_small_halo1", "jacobi", spec((96, 80, 72), halo=1.0), [7, 8, 13], GC),
    ("aniso_jacobi", "jacobi", spec((250, 34, 18)), [6], JC),
    ("aniso_gsn", "gs-naive", spec((250, 34, 18)), [3], GC),
]

# BASELINE config 4 (the bench's headline): weak-scaling 1024^3 per GPU and the
# strong-scaling 1024 x 1024 x 2048 grid, 100 sweeps.  ``--huge``: ~5 + ~10
# minutes on 8 cores with the reference's threaded k-slab engine; the 2048
# case peaks at ~52 GB of host memory (grid, uniform temp / scratch copy).
HUGE = [
    ("cfg4_jacobi1024", "jacobi", spec((1024, 1024, 1024)), [100], GC),
    ("cfg4_jacobi1024x2048", "jacobi", spec((1024, 1024, 2048)), [100], GC),
]

BIG = [
    ("cfg3_jacobi512_halo1", "jacobi", spec((512, 512, 512), halo=1.0), [4, 100], GC),
    ("cfg5_gsn512_mixed", "gs-naive", spec((512, 512, 512), lo=-1.0, hi=1.0), [100], GC),
    ("cfg5_gsi512_mixed", "gs-interleaved", spec((512, 512, 512), lo=-1.0, hi=1.0), [100], GC),
]


def samples(a):
    flat = a.ravel()
    idx = np.linspace(0, flat.size - 1, 16).astype(np.int64)
    return {"index": idx.tolist(), "value": [float(v).hex() for v in flat[idx]]}


def hashed_records(items, threads):
    out = {}
    for name, kernel, sp, iters_list, coeffs in items:
        for iters in iters_list:
            t0 = time.time()
            # the threaded/pipeline reference engines are bitwise equal to
            # run_serial (reference tests/test_sweeps_threaded.py); use them
            # for the large cases to keep generation time down
            if threads > 1 and sp["shape"][2] >= threads and sp["shape"][1] >= threads \
                    and np.prod(sp["shape"]) >= 64 ** 3:
                in_hash, got = ref_result(kernel, sp, iters, coeffs, variant="threaded",
                                          threads=threads)
            else:
                in_hash, got = ref_result(kernel, sp, iters, coeffs)
            key = f"{name}_it{iters}"
            out[key] = {"kernel": kernel, "spec": sp, "iters": iters,
                        "coeffs": [float(c).hex() for c in coeffs],
                        "input_sha256": in_hash, "output_sha256": sha(got),
                        "samples": samples(got)}
            print(f"{key}: {time.time() - t0:.1f}s", flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true")
    ap.add_argument("--huge", action="store_true",
                    help="only the config-4 records (skips the small cases)")
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    args = ap.parse_args()
    assert HAVE_NUMBA, "generate with the reference's compiled kernels"
    hpath = HERE / "hashes.json"
    if args.huge:
        hashes = json.loads(hpath.read_text())
        for name, kernel, sp, iters, coeffs in HUGE:
            hashes.update(hashed_records([(name, kernel, sp, iters, coeffs)], args.threads))
            hpath.write_text(json.dumps(hashes, indent=1, sort_keys=True))
        print(f"wrote {len(hashes)} hashed cases")
        return

    arrays, meta = {}, {}
    for name, kernel, sp, iters, coeffs in SMALL:
        in_hash, got = ref_result(kernel, sp, iters, coeffs)
        # cross-check with the reference's independent scalar oracle
        if np.prod(sp["shape"]) <= 20 ** 3:
            want = scalar_ref.run_reference(kernel, make_input(sp), coeffs[0], coeffs[1], iters)
            assert np.array_equal(got.ravel(), np.array(want)), name
        arrays[name] = got
        meta[name] = {"kernel": kernel, "spec": sp, "iters": iters,
                      "coeffs": [float(c).hex() for c in coeffs], "input_sha256": in_hash}
    np.savez_compressed(HERE / "small_cases.npz", **arrays)
    (HERE / "small_cases.json").write_text(json.dumps(meta, indent=1, sort_keys=True))
    print(f"wrote {len(arrays)} small cases")

    hashes = json.loads(hpath.read_text()) if hpath.exists() else {}
    hashes.update(hashed_records(HASHED, args.threads))
    if args.big:
        hashes.update(hashed_records(BIG, args.threads))
    hpath.write_text(json.dumps(hashes, indent=1, sort_keys=True))
    print(f"wrote {len(hashes)} hashed cases")


if __name__ == "__main__":
    main()
