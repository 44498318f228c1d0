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
The result is always left in ``g.data`` and ``g`` is returned.
"""

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
    return _finish(plan, g, stats, depth=depth, **extra)


def run_serial(plan, g, stats=None):
    """reference sweeps/serial.py:8-42 (the result is left in g)."""
    return _run(plan, g, stats)


def run_threaded_jacobi(plan, g, placement=None, stats=None):
    """reference sweeps/threaded.py:28-59: same checks; z-slab parallelism
    is the CTA grid (and the multi-GPU slab engine)."""
    if plan.kernel != JACOBI:
        raise PlanError(f"threaded engine is Jacobi-only, got kernel {plan.kernel!r}")
    if plan.threads > g.nk:
        raise PartitionError(f"{plan.threads} threads cannot split nk={g.nk} planes")
    return _run(plan, g, stats, pinned=None)


def run_pipeline_gs(plan, g, placement=None, stats=None):
    """reference sweeps/threaded.py:62-96: exact lexicographic order, here
    as the flag-pipelined tile wavefront."""
    if plan.kernel == JACOBI:
        raise PlanError("pipeline engine applies to Gauss-Seidel kernels only")
    if plan.threads > g.nj:
        raise PartitionError(f"{plan.threads} threads cannot split nj={g.nj} lines")
    out = _run(plan, g, stats, pinned=None)
    if stats is not None and plan.iter_end:
        stats["stages_per_sweep"] = g.nk + plan.threads - 1
    return out


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


def run(plan, g, placement=None, stats=None, instrument=False):
    """reference sweeps/__init__.py:52-71: variant dispatch; a GS kernel on
    the threaded variant runs the pipeline engine."""
    if plan.variant == SERIAL:
        return run_serial(plan, g, stats=stats)
    if plan.variant == THREADED:
        if plan.kernel == JACOBI:
            return run_threaded_jacobi(plan, g, placement=placement, stats=stats)
        return run_pipeline_gs(plan, g, placement=placement, stats=stats)
    if plan.variant == PIPELINE:
        return run_pipeline_gs(plan, g, placement=placement, stats=stats)
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
