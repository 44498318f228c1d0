"""Multi-GPU through the drop-in entry points (run / run_threaded_jacobi /
run_pipeline_gs with `devices`, C entry sb_run_multi): z-slabs for Jacobi
(reference sweeps/threaded.py:28-59, partition_blocks(nk, P) at :39) and the
cross-GPU z-pipeline for Gauss-Seidel (:62-96).  One GPU is visible, so the
slabs share it (devices=[0, 0, ...]) -- the same scatter, ghost exchange
and gather code as on several GPUs.  Bitwise against the reference's own
results (tests/golden) and the returned-grid contract of the reference's
ping-pong engines (serial.py:24-31: odd iter_end returns the copy)."""

import numpy as np
import pytest

import oracle
from conftest import coeffs_of, make_input, sha

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (run under gpurun)")


from paper_1004_1741_b200 import _lib  # noqa: E402
from paper_1004_1741_b200.errors import PartitionError  # noqa: E402
from paper_1004_1741_b200.kernels import JACOBI, StencilCoeffs  # noqa: E402
from paper_1004_1741_b200.sweeps import SweepPlan, run  # noqa: E402


def _plan(rec, a, b, variant="threaded"):
    return SweepPlan(rec["kernel"], variant, rec["iters"], threads=1, coeffs=StencilCoeffs(a, b))


@pytest.mark.parametrize("nslabs", [2, 3])
def test_small_cases_over_slabs_host_grids(small_cases, nslabs):
    """Every reference fixture with nk >= nslabs through run(threaded,
    devices=[0]*nslabs) on numpy grids."""
    checked = 0
    for name, (rec, want) in small_cases.items():
        a, b = coeffs_of(rec)
        g = make_input(rec["spec"])
        if g.nk < nslabs:
            with pytest.raises(PartitionError):
                run(_plan(rec, a, b), g, devices=[0] * nslabs)
            continue
        stats = {}
        out = run(_plan(rec, a, b), g, devices=[0] * nslabs, stats=stats)
        assert sha(out.data) == sha(want), (name, nslabs)
        assert stats["line_updates"] == rec["iters"] * g.nk * g.nj
        assert rec["iters"] == 0 or stats["slabs"] == nslabs
        checked += 1
    assert checked > 10


def test_device_grid_over_slabs(small_cases):
    """A CUDA-tensor grid is scattered from / gathered to device memory."""
    for name, (rec, want) in list(small_cases.items())[:12]:
        a, b = coeffs_of(rec)
        g = make_input(rec["spec"])
        if g.nk < 2:
            continue
        d = g.to_device("cuda:0")
        out = run(_plan(rec, a, b), d, devices=[0, 0])
        assert sha(out.data.cpu().numpy()) == sha(want), name


def test_environment_selects_the_devices(small_cases, monkeypatch):
    name, (rec, want) = next((n, v) for n, v in small_cases.items()
                             if v[0]["kernel"] == JACOBI and v[0]["spec"]["shape"][2] >= 4)
    a, b = coeffs_of(rec)
    monkeypatch.setenv("SB200_DEVICES", "0,0,0,0")
    stats = {}
    out = run(_plan(rec, a, b), make_input(rec["spec"]), stats=stats)
    assert stats["slabs"] == 4 and sha(out.data) == sha(want)


@pytest.mark.parametrize("kernel", ["gs-naive", "gs-interleaved"])
def test_gs_pipeline_over_slabs_vs_oracle(kernel):
    """Mixed-sign data, uneven slabs (nk = 23 over 4), 7 sweeps."""
    from paper_1004_1741_b200.grid import InitPattern, create_grid

    g = create_grid(34, 20, 23, InitPattern.seeded_random(5, -1.0, 1.0))
    want = oracle.run_serial(kernel, g.data.copy(), 7, 0.0, 1 / 6)
    stats = {}
    out = run(SweepPlan(kernel, "pipeline", 7, threads=3), g, devices=[0, 0, 0, 0], stats=stats)
    assert out is g and np.array_equal(out.data, want)
    assert stats["stages_per_sweep"] == 4


@pytest.mark.parametrize("variant", ["serial", "threaded"])
def test_odd_iterations_return_the_copy(variant):
    """reference serial.py:24-31 / threaded.py:59: for odd iter_end the
    returned grid is the scratch copy with the final field and g holds the
    field after iter_end - 1 sweeps; even iter_end returns g."""
    from paper_1004_1741_b200.grid import InitPattern, create_grid

    for n in (1, 5, 6):
        g = create_grid(18, 12, 10, InitPattern.seeded_random(9))
        base = g.data.copy()
        kw = {"devices": [0, 0]} if variant == "threaded" else {}
        out = run(SweepPlan("jacobi", variant, n, threads=2, coeffs=StencilCoeffs(0.25, 0.125)), g,
                  **kw)
        assert np.array_equal(out.data, oracle.run_serial("jacobi", base.copy(), n, 0.25, 0.125))
        if n % 2:
            assert out is not g
            prev = oracle.run_serial("jacobi", base.copy(), n - 1, 0.25, 0.125) if n > 1 else base
            assert np.array_equal(g.data, prev)
        else:
            assert out is g


def test_config4_strong_through_run_vs_reference_hash(hashed_cases):
    """BASELINE config 4 strong (1024 x 1024 x 2048, 100 sweeps) through the
    drop-in call a reference user makes -- run(threaded plan, numpy grid) --
    spread over two slabs: equals the reference's own result."""
    rec = hashed_cases["cfg4_jacobi1024x2048_it100"]
    a, b = coeffs_of(rec)
    g = make_input(rec["spec"])
    assert sha(g.data) == rec["input_sha256"]
    out = run(SweepPlan("jacobi", "threaded", rec["iters"], threads=8, coeffs=StencilCoeffs(a, b)),
              g, devices=[0, 0])
    assert sha(out.data) == rec["output_sha256"]
    _lib.release_caches(0)


def test_more_slabs_than_one_launch_takes_and_bad_devices():
    """9 GS slabs on one GPU exceed one fused launch (8): the launch-per-
    sweep pipeline runs instead, same bits; an invisible device index is a
    ValueError before any work."""
    from paper_1004_1741_b200.grid import InitPattern, create_grid

    g = create_grid(20, 18, 27, InitPattern.seeded_random(8, -1.0, 1.0))
    want = oracle.run_serial("gs-naive", g.data.copy(), 4, 0.0, 1 / 6)
    out = run(SweepPlan("gs-naive", "pipeline", 4), g, devices=[0] * 9)
    assert np.array_equal(out.data, want)
    h = create_grid(20, 18, 27, InitPattern.seeded_random(8))
    before = h.data.copy()
    with pytest.raises(ValueError):
        run(SweepPlan("jacobi", "threaded", 2), h, devices=[0, torch.cuda.device_count() + 3])
    assert np.array_equal(h.data, before)
