"""Host-side logic of the drop-in, restating the reference's own unit tests
(pkg/tests/test_plan.py, test_grid.py, test_sweeps_*.py argument checks)."""

import hashlib
import struct

import numpy as np
import pytest

from paper_1004_1741_b200.errors import (
    BoundsError,
    ConfigError,
    DimensionError,
    PartitionError,
    PlanError,
)
from paper_1004_1741_b200.grid import InitPattern, create_grid, dump_binary, flat_index, summary
from paper_1004_1741_b200.kernels import StencilCoeffs
from paper_1004_1741_b200.sweeps import (
    SweepPlan,
    WavefrontConfig,
    partition_blocks,
    run,
    run_batch,
    run_pipeline_gs,
    run_threaded_jacobi,
    run_wavefront,
    run_wavefront_gs,
    run_wavefront_jacobi,
)


def test_partition_reference_examples():
    assert partition_blocks(200, 8) == [(i * 25, (i + 1) * 25) for i in range(8)]
    assert partition_blocks(10, 3) == [(0, 4), (4, 7), (7, 10)]
    for bad in ((4, 5), (4, 0)):
        with pytest.raises(PartitionError):
            partition_blocks(*bad)


def test_partition_properties_exhaustive():
    for n in range(1, 65):
        for b in range(1, n + 1):
            r = partition_blocks(n, b)
            sizes = [hi - lo for lo, hi in r]
            assert len(r) == b and r[0][0] == 0 and r[-1][1] == n
            assert min(sizes) >= 1 and max(sizes) - min(sizes) <= 1
            assert sizes == sorted(sizes, reverse=True)
            assert all(x[1] == y[0] for x, y in zip(r, r[1:]))


def test_plan_validation():
    with pytest.raises(PlanError):
        SweepPlan("bogus", "serial", 1)
    with pytest.raises(PlanError):
        SweepPlan("jacobi", "bogus", 1)
    with pytest.raises(PlanError):
        SweepPlan("jacobi", "serial", -1)
    with pytest.raises(PlanError):
        SweepPlan("jacobi", "wavefront", 4)  # no config
    with pytest.raises(PlanError):
        SweepPlan("jacobi", "wavefront", 3, config=WavefrontConfig(1, 2, 2))
    with pytest.raises(PlanError):
        SweepPlan("jacobi", "wavefront", 3, config=WavefrontConfig(1, 3, 3))  # odd t > 1
    SweepPlan("gs-naive", "wavefront", 3, config=WavefrontConfig(1, 3, 3))  # odd t fine for GS
    with pytest.raises(PlanError):
        SweepPlan("jacobi", "pipeline", 1)
    with pytest.raises(PlanError):
        SweepPlan("gs-naive", "threaded", 1, threads=0)
    p = SweepPlan("jacobi", "serial", 2)
    assert (p.coeffs.a, p.coeffs.b) == (0.0, 1.0 / 6.0) and not p.is_gs


def test_wavefront_config_validation():
    for args in ((0, 1, 1), (1, 0, 1), (2, 1, 1)):
        with pytest.raises(ConfigError):
            WavefrontConfig(*args)
    with pytest.raises(ConfigError):
        WavefrontConfig(1, 2, 2, temp_planes=3)
    c = WavefrontConfig(2, 4, 8)
    assert c.temp_planes == 8 and c.total_threads == 8


def test_coeffs_must_be_finite():
    with pytest.raises(ValueError):
        StencilCoeffs(float("nan"), 0.1)
    with pytest.raises(ValueError):
        StencilCoeffs(0.1, float("inf"))


def test_engine_argument_errors_before_any_work():
    g = create_grid(4, 4, 4, InitPattern.seeded_random(1))
    with pytest.raises(PartitionError):
        run_threaded_jacobi(SweepPlan("jacobi", "threaded", 1, threads=5), g)
    with pytest.raises(PlanError):
        run_threaded_jacobi(SweepPlan("gs-naive", "threaded", 1, threads=2), g)
    with pytest.raises(PartitionError):
        run_pipeline_gs(SweepPlan("gs-naive", "pipeline", 1, threads=5), g)
    with pytest.raises(PartitionError):
        run_wavefront(SweepPlan("jacobi", "wavefront", 2, config=WavefrontConfig(1, 2, 40)), g)
    jplan = SweepPlan("jacobi", "wavefront", 2, config=WavefrontConfig(1, 2, 2))
    gplan = SweepPlan("gs-naive", "wavefront", 2, config=WavefrontConfig(1, 2, 2))
    with pytest.raises(PlanError):
        run_wavefront_jacobi(gplan, g)
    with pytest.raises(PlanError):
        run_wavefront_gs(jplan, g)


def test_run_batch_validates_before_any_work():
    """run_batch applies run()'s checks to every grid before touching a
    device (these raise on a CPU-only host)."""
    g = create_grid(4, 4, 4, InitPattern.seeded_random(1))
    h = create_grid(4, 4, 6, InitPattern.seeded_random(2))
    with pytest.raises(PartitionError):
        run_batch(SweepPlan("jacobi", "threaded", 1, threads=5), [g])
    with pytest.raises(PlanError):
        run_batch(SweepPlan("jacobi", "pipeline", 1), [g])
    with pytest.raises(PartitionError):
        run_batch(SweepPlan("jacobi", "wavefront", 2, config=WavefrontConfig(1, 2, 40)), [g])
    with pytest.raises(ValueError):
        run_batch(SweepPlan("jacobi", "serial", 1), [g, h])
    assert run_batch(SweepPlan("jacobi", "serial", 1), []) == []
    before = g.data.copy()
    assert run_batch(SweepPlan("jacobi", "serial", 0), [g])[0] is g
    assert np.array_equal(g.data, before)


def test_zero_iterations_return_the_grid_untouched():
    g = create_grid(5, 5, 5, InitPattern.seeded_random(42))
    before = g.data.copy()
    stats = {}
    out = run(SweepPlan("jacobi", "serial", 0), g, stats=stats)
    assert out is g and np.array_equal(g.data, before) and stats["line_updates"] == 0


def test_grid_patterns():
    g = create_grid(2, 2, 2, InitPattern.linear())
    assert g.data[1, 1, 1] == 0.0 and g.data[2, 2, 2] == 3.0 and g.data[0, 0, 0] == -3.0
    g = create_grid(3, 5, 7, InitPattern.uniform(1.5))
    assert g.data.size == 5 * 7 * 9 and np.all(g.data == 1.5)
    g = create_grid(4, 5, 6, InitPattern.seeded_random(7))
    halo = g.data.copy()
    halo[1:-1, 1:-1, 1:-1] = 0.0
    assert np.all(halo == 0.0) and g.interior.min() >= 0.0 and g.interior.max() < 1.0
    g = create_grid(4, 4, 4, InitPattern.seeded_random(1, lo=-2.0, hi=2.0))
    assert g.interior.min() >= -2.0 and g.interior.max() < 2.0
    assert g.data.ctypes.data % 64 == 0
    for bad in ((0, 1, 1), (1, -1, 1), (1.5, 1, 1)):
        with pytest.raises(DimensionError):
            create_grid(*bad, InitPattern.uniform(0))
    with pytest.raises(ValueError):
        InitPattern("bogus")


def test_flat_index_bijection_and_bounds():
    g = create_grid(3, 4, 5, InitPattern.uniform(0))
    seen = {flat_index(g, k, j, i) for k in range(-1, 6) for j in range(-1, 5) for i in range(-1, 4)}
    assert seen == set(range(g.data.size))
    with pytest.raises(BoundsError):
        flat_index(g, 6, 0, 0)


def test_dump_binary_and_summary(tmp_path):
    g = create_grid(3, 4, 5, InitPattern.seeded_random(3))
    p = tmp_path / "g.bin"
    dump_binary(g, p)
    raw = p.read_bytes()
    assert struct.unpack("<qqq", raw[:24]) == (3, 4, 5)
    assert np.array_equal(np.frombuffer(raw[24:], "<f8").reshape(5, 4, 3), g.interior)
    digest = hashlib.sha256(np.ascontiguousarray(g.interior).tobytes()).hexdigest()[:16]
    assert summary(g).endswith(f"sha256[:16]={digest}")


def test_line_api_argument_errors_without_device():
    from paper_1004_1741_b200.errors import AliasingError, ShapeError
    from paper_1004_1741_b200.kernels import gs_line_update, jacobi_line_update

    src = create_grid(6, 6, 6, InitPattern.seeded_random(1))
    with pytest.raises(ShapeError):
        jacobi_line_update(src, create_grid(5, 6, 6, InitPattern.uniform(0)), StencilCoeffs(0, 0.1), 0, 0)
    with pytest.raises(AliasingError):
        jacobi_line_update(src, src, StencilCoeffs(0, 0.1), 0, 0)
    with pytest.raises(BoundsError):
        jacobi_line_update(src, create_grid(6, 6, 6, InitPattern.uniform(0)), StencilCoeffs(0, 0.1), 6, 0)
    with pytest.raises(BoundsError):
        gs_line_update(src, 0.1, 0, -1)


def test_resolve_devices_forms(monkeypatch):
    from paper_1004_1741_b200.sweeps.engine import resolve_devices

    monkeypatch.delenv("SB200_DEVICES", raising=False)
    assert resolve_devices() is None
    assert resolve_devices(3) == [0, 1, 2]
    assert resolve_devices([2, 0, 2]) == [2, 0, 2]
    assert resolve_devices("1,3") == [1, 3]
    assert resolve_devices("2") == [0, 1]
    monkeypatch.setenv("SB200_DEVICES", "0,0,1")
    assert resolve_devices() == [0, 0, 1]
    assert resolve_devices([5]) == [5]  # explicit argument wins over the environment
    for bad in (0, [], "0,"[:0] or "-1"):
        with pytest.raises(ValueError):
            resolve_devices(bad)


def test_multi_gpu_argument_errors_before_any_work(monkeypatch):
    """More GPUs than planes is the reference's PartitionError for P > nk
    (threaded.py:31-33), raised before a device is touched."""
    monkeypatch.delenv("SB200_DEVICES", raising=False)
    g = create_grid(4, 4, 3, InitPattern.seeded_random(1))
    with pytest.raises(PartitionError):
        run(SweepPlan("jacobi", "threaded", 2, threads=2), g, devices=[0, 0, 0, 0])
    with pytest.raises(PartitionError):
        run(SweepPlan("gs-naive", "pipeline", 2, threads=2), g, devices=4)
    monkeypatch.setenv("SB200_DEVICES", "0,0,0,0")
    with pytest.raises(PartitionError):
        run_threaded_jacobi(SweepPlan("jacobi", "threaded", 2), g)
    with pytest.raises(PlanError):
        run_pipeline_gs(SweepPlan("jacobi", "pipeline", 2), g)


def test_barrier_phase_counts():
    from paper_1004_1741_b200.sweeps.engine import barrier_phases, gs_stages_per_sweep

    assert barrier_phases(SweepPlan("jacobi", "serial", 0), 4) == 0
    assert barrier_phases(SweepPlan("jacobi", "serial", 100), 4) == 25
    assert barrier_phases(SweepPlan("jacobi", "serial", 10), 3) == 4
    assert barrier_phases(SweepPlan("jacobi", "serial", 16), 8) == 4  # passes of at most 4
    assert barrier_phases(SweepPlan("gs-naive", "serial", 100), 1) == 1
    g = create_grid(8, 40, 30, InitPattern.uniform(0))
    assert gs_stages_per_sweep(g, 100) == 3 + 5 - 1
    assert gs_stages_per_sweep(g, 1) == 3 + 2 - 1


def test_seeded_planes_equal_create_grid_slices():
    from paper_1004_1741_b200.grid import seeded_planes

    for (ni, nj, nk), (lo, hi) in (((7, 5, 9), (0.0, 1.0)), ((4, 6, 3), (-1.0, 1.0))):
        full = create_grid(ni, nj, nk, InitPattern.seeded_random(42, lo, hi)).data
        for p_lo, p_hi in ((0, nk + 2), (0, 1), (1, 4), (2, nk + 2), (nk + 1, nk + 2), (3, 3)):
            got = seeded_planes(42, ni, nj, nk, p_lo, p_hi, lo, hi)
            assert got.tobytes() == full[p_lo:p_hi].tobytes(), (ni, nj, nk, p_lo, p_hi)
    with pytest.raises(BoundsError):
        seeded_planes(42, 3, 3, 3, 2, 6)


def test_multi_gpu_path_reaches_the_library_without_a_gpu(monkeypatch):
    """On a CPU-only host the multi-GPU drop-in path fails loudly at the
    device check (no CPU fallback) -- after all argument handling."""
    import torch

    from paper_1004_1741_b200.errors import DeviceError

    if torch.cuda.is_available():
        pytest.skip("CPU-only check")
    monkeypatch.delenv("SB200_DEVICES", raising=False)
    g = create_grid(4, 4, 6, InitPattern.seeded_random(1))
    for plan in (SweepPlan("jacobi", "threaded", 3, threads=2), SweepPlan("gs-naive", "pipeline", 2)):
        with pytest.raises(DeviceError):
            run(plan, g, devices=[0, 0])
