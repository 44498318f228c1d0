"""GPU sweep engines behind the reference's entry points.

Every reference engine (serial, threaded, pipeline, wavefront; reference
pkg/src/stencilbench/sweeps/{serial,threaded,wavefront}.py) computes the
same bits -- the reference pins that with its own equivalence tests -- so
on the B200 they all run the same device code: the temporally blocked
Jacobi kernel (depth = the plan's wavefront t, else DEFAULT_DEPTH) or the
flag-pipelined lexicographic Gauss-Seidel kernel.  What the variants still
contribute is their contract: argument validation and exceptions
(raised before any work, like the reference), the returned grid, and the
``stats`` keys.

Grids: ``g.data`` as a host numpy array goes through ``sb_run_host`` (copy
in, sweep, copy out; synchronous).  As a CUDA float64 torch tensor it is
swept in place on the current stream through ``sb_jacobi`` / ``sb_gs``.

Returned grid (reference sweeps/serial.py:24-31, threaded.py:41-59): the
serial and threaded Jacobi engines ping-pong ``g`` and ``g.copy()``, so for
an odd ``iter_end`` they return the copy holding the final field and leave
``g`` at sweep ``iter_end - 1``; every other engine returns ``g`` itself.

Several GPUs: the threaded engines (``run_threaded_jacobi``, and
``run_pipeline_gs`` for the GS kernels) take ``devices`` -- a sequence of
CUDA device indices, an int N (the first N GPUs) or "all"; default the
``SB200_DEVICES`` environment variable (same forms), else one GPU.  With
more than one device the grid is cut into z-slabs (the reference's
``partition_blocks(nk, P)`` k-slabs, threaded.py:39), one per device, and
runs through ``sb_run_multi``: Jacobi with per-time-block halo exchange,
GS as the exact cross-GPU z-pipeline.  Bitwise equal to one GPU.
"""

import os

import ctypes

import numpy as np

from .. import _lib
from ..errors import PartitionError, PlanError
from ..kernels import JACOBI
from .plan import PIPELINE, SERIAL, THREADED, WAVEFRONT, partition_blocks

# Temporal block depth used when the plan does not name one (variants other
# than wavefront).  Results do not depend on it; throughput does.
DEFAULT_DEPTH = 4

_scratch_cache = {}


def _is_torch(x):
    return type(x).__module__.startswith("torch")


def resolve_depth(plan, g):
    """Sweeps fused per HBM pass for a Jacobi plan."""
    if plan.kernel != JACOBI:
        return 1
    if plan.variant == WAVEFRONT and plan.config is not None:
        depth = plan.config.threads_per_group
    else:
        depth = DEFAULT_DEPTH
    # (odd ni: the library runs the fused depths on pitched copies)
    return max(1, min(depth, _lib.max_depth()))


def _scratch_for(t):
    import torch

    key = (t.device, tuple(t.shape))
    buf = _scratch_cache.get(key)
    if buf is None:
        _scratch_cache.clear()  # keep at most one scratch grid alive
        buf = torch.empty_like(t, memory_format=torch.contiguous_format)
        _scratch_cache[key] = buf
    return buf


def execute(kernel, g, iters, a, b, depth, sync=True):
    """Run `iters` sweeps of `kernel` on g in place (device code only)."""
    lib = _lib.load()
    _lib.require_device()
    kid = _lib.KERNEL_IDS[kernel]
    data = g.data
    if _is_torch(data):
        import torch

        if not data.is_cuda or data.dtype != torch.float64 or not data.is_contiguous():
            raise ValueError("device grids must be contiguous float64 CUDA tensors")
        if tuple(data.shape) != g.shape_padded:
            raise ValueError(f"grid data shape {tuple(data.shape)} != {g.shape_padded}")
        with torch.cuda.device(data.device):
            stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
            if kernel == JACOBI:
                scratch = _scratch_for(data)
                in_s = ctypes.c_int(0)
                _lib.check(lib.sb_jacobi(data.data_ptr(), scratch.data_ptr(), g.ni, g.nj, g.nk,
                                         iters, a, b, depth, stream, ctypes.byref(in_s)))
                if in_s.value:
                    data.copy_(scratch)
            else:
                _lib.check(lib.sb_gs(data.data_ptr(), g.ni, g.nj, g.nk, iters, b, kid, stream))
            if sync:
                _lib.check(lib.sb_sync(stream))
        return g
    arr = data
    if not (isinstance(arr, np.ndarray) and arr.dtype == np.float64 and arr.flags.c_contiguous
            and arr.flags.writeable):
        raise ValueError("host grids must be writeable C-contiguous float64 numpy arrays")
    if arr.shape != g.shape_padded:
        raise ValueError(f"grid data shape {arr.shape} != {g.shape_padded}")
    device = 0
    try:
        import torch

        if torch.cuda.is_available():
            device = torch.cuda.current_device()
    except ImportError:
        pass
    _lib.check(lib.sb_run_host(kid, arr.ctypes.data, g.ni, g.nj, g.nk, iters, a, b, depth, device))
    return g


def resolve_devices(devices=None):
    """GPUs for the threaded engines: a list of CUDA device indices, or None
    for the single-GPU path.  `devices`: a sequence of indices, an int N (the
    first N visible GPUs) or "all"; None reads $SB200_DEVICES ("0,1,2,3",
    "4" or "all")."""
    if devices is None:
        env = os.environ.get("SB200_DEVICES", "").strip()
        if not env:
            return None
        devices = env
    if isinstance(devices, str):
        text = devices.strip().lower()
        if text == "all":
            devices = _lib.device_count()
        elif "," in text:
            devices = [int(x) for x in text.split(",") if x.strip()]
        else:
            devices = int(text)
    if isinstance(devices, int):
        if devices < 1:
            raise ValueError(f"need at least one GPU, got {devices}")
        return list(range(devices))
    out = [int(d) for d in devices]
    if not out:
        raise ValueError("empty device list")
    return out


def barrier_phases(plan, depth):
    """Device-wide synchronisation points of the GPU run -- the counterpart
    of the reference wavefront engines' stats["barrier_phases"] (one barrier
    per plane phase, wavefront.py:308-311): kernel-launch boundaries.  A
    Jacobi run is ceil(iter_end / depth) fused launches (passes); a GS run
    is one launch per call (its sweeps are pipelined inside)."""
    if plan.iter_end == 0:
        return 0
    if plan.kernel != JACOBI:
        return 1
    eff = depth if depth <= 4 else 4  # sb_jacobi fuses at most 4 per pass
    return -(-plan.iter_end // eff)


def _finish(plan, g, stats, **extra):
    if stats is not None:
        stats["line_updates"] = plan.iter_end * g.nk * g.nj
        stats["engine"] = "b200"
        stats.update(extra)
    return g


def _run(plan, g, stats, **extra):
    if plan.iter_end == 0:
        if stats is not None:
            stats["line_updates"] = 0
        return g
    depth = resolve_depth(plan, g)
    execute(plan.kernel, g, plan.iter_end, plan.coeffs.a, plan.coeffs.b, depth)
    return _finish(plan, g, stats, depth=depth, barrier_phases=barrier_phases(plan, depth), **extra)


def _run_pingpong(plan, g, stats, devs=None, **extra):
    """Jacobi engines that own two grids (serial, threaded): for an odd
    iter_end the final field is returned in a new grid (the reference's
    g.copy()) and g holds sweep iter_end - 1."""
    n = plan.iter_end
    if n == 0:
        if stats is not None:
            stats["line_updates"] = 0
        return g
    depth = resolve_depth(plan, g)
    sweep = (lambda grid, k: _execute_multi(plan.kernel, grid, k, plan.coeffs.a, plan.coeffs.b,
                                            depth, devs)) if devs else \
        (lambda grid, k: execute(plan.kernel, grid, k, plan.coeffs.a, plan.coeffs.b, depth))
    out = g
    if n % 2 == 0:
        sweep(g, n)
    else:
        if n > 1:
            sweep(g, n - 1)
        out = g.copy()
        sweep(out, 1)
    phases = barrier_phases(plan, depth) + (1 if n % 2 and n > 1 else 0)
    _finish(plan, g, stats, depth=depth, barrier_phases=phases, **extra)
    return out


def _execute_multi(kernel, g, iters, a, b, depth, devices):
    """`iters` sweeps of g across `devices` (z-slabs, sb_run_multi); g may
    be a host numpy grid or a CUDA tensor on any device.  Synchronous."""
    lib = _lib.load()
    _lib.require_device()
    data = g.data
    if _is_torch(data):
        import torch

        if not data.is_cuda or data.dtype != torch.float64 or not data.is_contiguous():
            raise ValueError("device grids must be contiguous float64 CUDA tensors")
        if tuple(data.shape) != g.shape_padded:
            raise ValueError(f"grid data shape {tuple(data.shape)} != {g.shape_padded}")
        torch.cuda.current_stream(data.device).synchronize()  # the library uses its own streams
        ptr = data.data_ptr()
    else:
        if not (isinstance(data, np.ndarray) and data.dtype == np.float64
                and data.flags.c_contiguous and data.flags.writeable):
            raise ValueError("host grids must be writeable C-contiguous float64 numpy arrays")
        if data.shape != g.shape_padded:
            raise ValueError(f"grid data shape {data.shape} != {g.shape_padded}")
        ptr = data.ctypes.data
    devs = (ctypes.c_int * len(devices))(*devices)
    _lib.check(lib.sb_run_multi(_lib.KERNEL_IDS[kernel], ptr, g.ni, g.nj, g.nk, iters, a, b,
                                depth, len(devices), devs))
    return g


def _multi(devices):
    devs = resolve_devices(devices)
    return devs if devs is not None and len(devs) > 1 else None


def run_serial(plan, g, stats=None):
    """reference sweeps/serial.py:8-42."""
    if plan.kernel == JACOBI:
        return _run_pingpong(plan, g, stats)
    return _run(plan, g, stats)


def run_threaded_jacobi(plan, g, placement=None, stats=None, devices=None):
    """reference sweeps/threaded.py:28-59: same checks and returned grid;
    z-slab parallelism is the CTA grid on one GPU, or z-slabs across
    `devices` (module docstring) with halo exchange between time blocks."""
    if plan.kernel != JACOBI:
        raise PlanError(f"threaded engine is Jacobi-only, got kernel {plan.kernel!r}")
    if plan.threads > g.nk:
        raise PartitionError(f"{plan.threads} threads cannot split nk={g.nk} planes")
    devs = _multi(devices)
    if devs is not None and len(devs) > g.nk:
        raise PartitionError(f"{len(devs)} GPUs cannot split nk={g.nk} planes")
    extra = {"pinned": None}
    if devs is not None:
        extra.update(devices=devs, slabs=len(devs))
    return _run_pingpong(plan, g, stats, devs, **extra)


def run_pipeline_gs(plan, g, placement=None, stats=None, devices=None):
    """reference sweeps/threaded.py:62-96: exact lexicographic order, here
    as the flag-pipelined tile wavefront on one GPU, or the cross-GPU
    z-pipeline of slabs over `devices`."""
    if plan.kernel == JACOBI:
        raise PlanError("pipeline engine applies to Gauss-Seidel kernels only")
    if plan.threads > g.nj:
        raise PartitionError(f"{plan.threads} threads cannot split nj={g.nj} lines")
    devs = _multi(devices)
    if devs is not None and len(devs) > g.nk:
        raise PartitionError(f"{len(devs)} GPUs cannot split nk={g.nk} planes")
    if plan.iter_end == 0:
        if stats is not None:
            stats["line_updates"] = 0
        return g
    if devs is None:
        out = _run(plan, g, stats, pinned=None)
        if stats is not None:
            stats["stages_per_sweep"] = gs_stages_per_sweep(g, plan.iter_end)
        return out
    _execute_multi(plan.kernel, g, plan.iter_end, 0.0, plan.coeffs.b, 1, devs)
    # z-pipeline: a sweep of G slabs takes G stages to pass through
    # (sweep s of slab g runs once slab g-1 finished sweep s)
    return _finish(plan, g, stats, depth=1, pinned=None, devices=devs, slabs=len(devs),
                   stages_per_sweep=len(devs), barrier_phases=plan.iter_end + len(devs) - 1)


def gs_stages_per_sweep(g, iters):
    """Hyperplane stages of one GS sweep on the GPU: tiles of 16 j-lines x
    BK k-planes (gs.cu: BK = 16 for calls of one or two sweeps, else 6) run
    along anti-diagonals J + K, so a sweep passes through
    tiles_j + tiles_k - 1 stages -- the counterpart of the reference
    pipeline's nk + P - 1 (threaded.py:81)."""
    bk = 16 if iters <= 2 else 6
    return -(-g.nj // 16) + -(-g.nk // bk) - 1


def _wavefront_checks(plan, g):
    cfg = plan.config
    if cfg is None:
        raise PlanError("wavefront engines need a plan with a WavefrontConfig")
    partition_blocks(g.nj, cfg.blocks)  # PartitionError when B > nj


def run_wavefront(plan, g, placement=None, stats=None, instrument=False):
    """reference sweeps/wavefront.py:127-131: temporal blocking with depth t."""
    _wavefront_checks(plan, g)
    return _run(plan, g, stats, pinned=None)


def run_wavefront_jacobi(plan, g, placement=None, stats=None, instrument=False):
    if plan.kernel != JACOBI:
        raise PlanError(f"jacobi wavefront engine got kernel {plan.kernel!r}")
    return run_wavefront(plan, g, placement, stats, instrument)


def run_wavefront_gs(plan, g, placement=None, stats=None, instrument=False):
    if plan.kernel == JACOBI:
        raise PlanError("gs wavefront engine needs a Gauss-Seidel kernel")
    return run_wavefront(plan, g, placement, stats, instrument)


def run(plan, g, placement=None, stats=None, instrument=False, devices=None):
    """reference sweeps/__init__.py:52-71: variant dispatch; a GS kernel on
    the threaded variant runs the pipeline engine.  `devices` (or
    $SB200_DEVICES) spreads the threaded/pipeline engines over GPUs."""
    if plan.variant == SERIAL:
        return run_serial(plan, g, stats=stats)
    if plan.variant == THREADED:
        if plan.kernel == JACOBI:
            return run_threaded_jacobi(plan, g, placement=placement, stats=stats, devices=devices)
        return run_pipeline_gs(plan, g, placement=placement, stats=stats, devices=devices)
    if plan.variant == PIPELINE:
        return run_pipeline_gs(plan, g, placement=placement, stats=stats, devices=devices)
    if plan.variant == WAVEFRONT:
        return run_wavefront(plan, g, placement=placement, stats=stats, instrument=instrument)
    raise PlanError(f"unknown variant {plan.variant!r}")


def _validate(plan, g):
    """The checks `run(plan, g)` performs before any work (same exceptions)."""
    if plan.variant in (THREADED, PIPELINE):
        if plan.kernel == JACOBI:
            if plan.variant == PIPELINE:
                raise PlanError("pipeline engine applies to Gauss-Seidel kernels only")
            if plan.threads > g.nk:
                raise PartitionError(f"{plan.threads} threads cannot split nk={g.nk} planes")
        elif plan.threads > g.nj:
            raise PartitionError(f"{plan.threads} threads cannot split nj={g.nj} lines")
    elif plan.variant == WAVEFRONT:
        _wavefront_checks(plan, g)
    elif plan.variant != SERIAL:
        raise PlanError(f"unknown variant {plan.variant!r}")


def run_batch(plan, grids, device=None):
    """`run(plan, g)` for each host grid of `grids` (one shape, numpy data),
    pipelined on one GPU through ``sb_run_host_batch``: grid i's upload
    overlaps grid i-1's sweeps and grid i-2's download.  Grids are processed
    in order and updated in place; every grid is validated first (same
    exceptions as `run`, raised before any work).  Returns `grids`."""
    grids = list(grids)
    if not grids:
        return grids
    g0 = grids[0]
    arrs = []
    for g in grids:
        _validate(plan, g)
        if (g.ni, g.nj, g.nk) != (g0.ni, g0.nj, g0.nk):
            raise ValueError("run_batch needs grids of one shape")
        arr = g.data
        if not (isinstance(arr, np.ndarray) and arr.dtype == np.float64 and arr.flags.c_contiguous
                and arr.flags.writeable and arr.shape == g.shape_padded):
            raise ValueError("run_batch needs writeable C-contiguous float64 host grids")
        arrs.append(arr)
    if plan.iter_end == 0:
        return grids
    lib = _lib.load()
    _lib.require_device()
    if device is None:
        import torch

        device = torch.cuda.current_device()
    ptrs = (ctypes.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
    depth = resolve_depth(plan, g0)
    _lib.check(lib.sb_run_host_batch(_lib.KERNEL_IDS[plan.kernel], ptrs, len(arrs), g0.ni, g0.nj,
                                     g0.nk, plan.iter_end, plan.coeffs.a, plan.coeffs.b, depth,
                                     device))
    return grids
