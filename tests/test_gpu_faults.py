"""Failure semantics on the GPU: a Gauss-Seidel launch whose inter-CTA
dependency never resolves is abandoned cooperatively and reported as
DeviceError (SB_ERR_TIMEOUT), and the CUDA context stays usable -- the next
call runs normally and matches the oracle.  The reference's counterpart is
the poisoned barrier + re-raise in the caller (reference sync.py:31-32,
sweeps/team.py:42-64); its test is pkg/tests/test_sync.py's poison case."""

import ctypes
import time

import numpy as np
import pytest

import oracle
from conftest import sha

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_1004_1741_b200 import _lib  # noqa: E402
from paper_1004_1741_b200.errors import DeviceError  # noqa: E402
from paper_1004_1741_b200.grid import InitPattern, create_grid  # noqa: E402


@pytest.fixture(autouse=True)
def _clear_fault():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (run under gpurun)")
    yield
    _lib.check(_lib.load().sb_debug_fault(0, 0))


def _gs(dev, iters, kid):
    lib = _lib.load()
    n = dev.shape[2] - 2, dev.shape[1] - 2, dev.shape[0] - 2
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    _lib.check(lib.sb_gs(dev.data_ptr(), *n, iters, 1 / 6, kid, st))
    _lib.check(lib.sb_sync(st))


@pytest.mark.parametrize("kernel", ["gs-naive", "gs-interleaved"])
def test_withheld_progress_times_out_and_context_survives(kernel):
    lib = _lib.load()
    kid = _lib.KERNEL_IDS[kernel]
    g = create_grid(200, 96, 80, InitPattern.seeded_random(7, -1.0, 1.0))
    dev = torch.from_numpy(g.data.copy()).cuda()
    # ~0.1 s without progress ends a wait; tile 0 withholds its sweep-0 progress
    _lib.check(lib.sb_debug_fault(1, 1 << 27))
    t0 = time.perf_counter()
    with pytest.raises(DeviceError, match="timed out"):
        _gs(dev, 6, kid)
    assert time.perf_counter() - t0 < 30
    # normal operation again: same context, result bitwise == oracle
    _lib.check(lib.sb_debug_fault(0, 0))
    dev = torch.from_numpy(g.data.copy()).cuda()
    _gs(dev, 6, kid)
    want = oracle.run_serial(kernel, g.data, 6)
    assert sha(dev.cpu().numpy()) == sha(want)
    # and the Jacobi path on the same context
    from paper_1004_1741_b200.sweeps import execute

    h = create_grid(64, 48, 40, InitPattern.seeded_random(3))
    d = h.to_device("cuda:0")
    execute("jacobi", d, 8, 0.0, 1 / 6, 4)
    assert sha(d.data.cpu().numpy()) == sha(oracle.run_serial("jacobi", h.data, 8))
