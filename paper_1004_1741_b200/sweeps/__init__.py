"""Sweep engines of the drop-in: the reference's entry points
(pkg/src/stencilbench/sweeps/__init__.py) over the B200 kernels."""

from .engine import (
    DEFAULT_DEPTH,
    execute,
    resolve_depth,
    run,
    run_batch,
    run_pipeline_gs,
    run_serial,
    run_threaded_jacobi,
    run_wavefront,
    run_wavefront_gs,
    run_wavefront_jacobi,
)
from .plan import (
    BARRIER_AUTO,
    PIPELINE,
    SERIAL,
    THREADED,
    VARIANTS,
    WAVEFRONT,
    SweepPlan,
    WavefrontConfig,
    partition_blocks,
)

__all__ = [
    "BARRIER_AUTO", "DEFAULT_DEPTH", "PIPELINE", "SERIAL", "THREADED", "VARIANTS", "WAVEFRONT",
    "SweepPlan", "WavefrontConfig", "execute", "partition_blocks", "resolve_depth", "run", "run_batch",
    "run_pipeline_gs", "run_serial", "run_threaded_jacobi", "run_wavefront", "run_wavefront_gs",
    "run_wavefront_jacobi",
]
