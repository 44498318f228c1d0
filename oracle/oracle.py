"""TEST INFRASTRUCTURE ONLY -- ctypes wrapper of the CPU oracle
(oracle/sb_oracle.c, a plain-C restatement of the reference sweeps).

Used by tests/ (as the parity checker), __graft_entry__.smoke() (checker)
and bench.py (cpu_baseline leg and ``--impl reference``).  The product
package never imports this module.

Pinned against the reference: tests/test_oracle.py compares every entry
point bit for bit with tests/golden/ (fixtures produced by the reference
package itself, tests/golden/make_golden.py).
"""

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "libsb_oracle.so"

KERNEL_IDS = {"jacobi": 0, "gs-naive": 1, "gs-interleaved": 2}

_lib = None


def build():
    subprocess.run(["make", "-C", str(HERE), "-s"], check=True)


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not LIB.exists():
        build()
    lib = ctypes.CDLL(str(LIB))
    i64, dbl, vp, i32 = ctypes.c_int64, ctypes.c_double, ctypes.c_void_p, ctypes.c_int
    lib.sbo_run_serial.argtypes = [i32, vp, vp, i64, i64, i64, i64, dbl, dbl]
    lib.sbo_run_serial.restype = i32
    lib.sbo_run_threaded_jacobi.argtypes = [vp, vp, i64, i64, i64, i64, dbl, dbl, i32]
    lib.sbo_run_threaded_jacobi.restype = i32
    lib.sbo_run_pipeline_gs.argtypes = [i32, vp, i64, i64, i64, i64, dbl, i32]
    lib.sbo_run_pipeline_gs.restype = i32
    lib.sbo_run_wavefront.argtypes = [i32, vp, i64, i64, i64, i64, dbl, dbl, i32, i32, i32]
    lib.sbo_run_wavefront.restype = i64
    for name in ("sbo_gs_window", "sbo_gs_window_interleaved"):
        getattr(lib, name).argtypes = [vp, vp, vp, i64, dbl, i64, i64]
        getattr(lib, name).restype = None
    _lib = lib
    return lib


def _check(arr):
    if not (arr.dtype == np.float64 and arr.flags.c_contiguous and arr.ndim == 3):
        raise ValueError("oracle grids are C-contiguous float64 (nk+2, nj+2, ni+2) arrays")
    nk, nj, ni = (s - 2 for s in arr.shape)
    return ni, nj, nk


def run_serial(kernel, data, iters, a=0.0, b=1.0 / 6.0):
    """Serial reference sweeps (sweeps/serial.py:8-42).  Returns a new array
    holding the final field; `data` is not modified."""
    g = np.array(data, dtype=np.float64, order="C", copy=True)
    ni, nj, nk = _check(g)
    scratch = np.empty_like(g) if kernel == "jacobi" else g
    in_s = load().sbo_run_serial(KERNEL_IDS[kernel], g.ctypes.data, scratch.ctypes.data,
                                 ni, nj, nk, iters, a, b)
    return scratch if in_s else g


def run_threaded(kernel, data, iters, a=0.0, b=1.0 / 6.0, threads=None):
    """Threaded Jacobi (k-slabs, threaded.py:28-59) or pipeline GS
    (j-blocks, threaded.py:62-96) on `threads` host threads.  Bitwise equal
    to run_serial.  Returns a new array holding the final field."""
    threads = threads or os.cpu_count() or 1
    g = np.array(data, dtype=np.float64, order="C", copy=True)
    ni, nj, nk = _check(g)
    lib = load()
    if kernel == "jacobi":
        threads = max(1, min(threads, nk))
        scratch = np.empty_like(g)
        in_s = lib.sbo_run_threaded_jacobi(g.ctypes.data, scratch.ctypes.data, ni, nj, nk, iters,
                                           a, b, threads)
        if in_s < 0:
            raise ValueError("partition error")
        return scratch if in_s else g
    threads = max(1, min(threads, nj))
    rc = lib.sbo_run_pipeline_gs(KERNEL_IDS[kernel], g.ctypes.data, ni, nj, nk, iters, b, threads)
    if rc < 0:
        raise ValueError("partition error")
    return g


def run_wavefront(kernel, data, iters, a=0.0, b=1.0 / 6.0, groups=1, tpg=2, blocks=None):
    """Wavefront temporal blocking (reference sweeps/wavefront.py:127-376):
    `groups` x `tpg` host threads, `blocks` j-blocks (default: groups).
    Returns (new array with the final field, barrier phases)."""
    g = np.array(data, dtype=np.float64, order="C", copy=True)
    ni, nj, nk = _check(g)
    blocks = blocks or groups
    phases = load().sbo_run_wavefront(KERNEL_IDS[kernel], g.ctypes.data, ni, nj, nk, iters, a, b,
                                      groups, tpg, blocks)
    if phases < 0:
        raise ValueError("plan error (iters % t, odd t for Jacobi, or blocks outside [1, nj])")
    return g, phases


def time_variant(kernel, variant, data, iters, a=0.0, b=1.0 / 6.0, threads=None, groups=None,
                 tpg=None, blocks=None):
    """Seconds spent in `iters` sweeps of `data` by one reference CPU engine
    (variant "threaded": k-slab Jacobi / pipeline GS on `threads`;
    "wavefront": `groups` x `tpg` threads over `blocks` j-blocks), setup
    excluded (working copies allocated and touched first) -- the CPU
    baseline legs of bench.py."""
    import time

    g = np.array(data, dtype=np.float64, order="C", copy=True)
    ni, nj, nk = _check(g)
    lib = load()
    kid = KERNEL_IDS[kernel]
    if variant == "wavefront":
        blocks = blocks or groups
        t0 = time.perf_counter()
        rc = lib.sbo_run_wavefront(kid, g.ctypes.data, ni, nj, nk, iters, a, b, groups, tpg, blocks)
    elif kernel == "jacobi":
        scratch = g.copy()
        threads = max(1, min(threads or os.cpu_count() or 1, nk))
        t0 = time.perf_counter()
        rc = lib.sbo_run_threaded_jacobi(g.ctypes.data, scratch.ctypes.data, ni, nj, nk, iters, a,
                                         b, threads)
    else:
        threads = max(1, min(threads or os.cpu_count() or 1, nj))
        t0 = time.perf_counter()
        rc = lib.sbo_run_pipeline_gs(kid, g.ctypes.data, ni, nj, nk, iters, b, threads)
    sec = time.perf_counter() - t0
    if rc < 0:
        raise ValueError("plan/partition error")
    return sec


def time_threaded_jacobi(data, iters, a=0.0, b=1.0 / 6.0, threads=None):
    """Seconds spent in `iters` threaded Jacobi sweeps of `data` (k-slabs,
    reference threaded.py:28-59), excluding the setup: the working copy and
    the scratch grid are allocated and touched first, so a short bounded
    sample measures the sweep rate rather than page faults (CPU baseline of
    bench.py)."""
    import time

    threads = threads or os.cpu_count() or 1
    g = np.array(data, dtype=np.float64, order="C", copy=True)
    ni, nj, nk = _check(g)
    scratch = g.copy()
    lib = load()
    threads = max(1, min(threads, nk))
    t0 = time.perf_counter()
    in_s = lib.sbo_run_threaded_jacobi(g.ctypes.data, scratch.ctypes.data, ni, nj, nk, iters, a, b,
                                       threads)
    sec = time.perf_counter() - t0
    if in_s < 0:
        raise ValueError("partition error")
    return sec


def gs_line(kernel, data, k, j, b):
    """One in-place GS line update of interior line (k, j) (reference
    kernels.py:236-247 via the window kernels).  Returns a new array."""
    g = np.array(data, dtype=np.float64, order="C", copy=True)
    ni, nj, nk = _check(g)
    fn = load().sbo_gs_window_interleaved if kernel == "gs-interleaved" else load().sbo_gs_window
    plane = (nj + 2) * (ni + 2) * 8
    base = g.ctypes.data
    fn(base + k * plane, base + (k + 1) * plane, base + (k + 2) * plane, ni + 2, b, j + 1, j + 2)
    return g
