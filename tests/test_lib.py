"""libsb200.so: loads, exports every symbol include/stencil_b200.h declares,
and rejects bad arguments before any device work (no GPU needed)."""

import ctypes
import re
from pathlib import Path

import pytest

from paper_1004_1741_b200 import _lib
from paper_1004_1741_b200.errors import DimensionError, PartitionError, PlanError

HEADER = Path(__file__).resolve().parent.parent / "include" / "stencil_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sb_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_abi():
    syms = declared_symbols()
    assert "sb_jacobi" in syms and "sb_gs" in syms and "sb_run_host" in syms
    assert set(syms) == set(_lib.SIGNATURES), "ctypes table out of sync with the header"


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_version_and_depth():
    lib = _lib.load()
    assert lib.sb_version() >= 100
    assert _lib.max_depth() == 8


def _jac(lib, ni=8, nj=8, nk=8, iters=1, depth=1, g=1 << 12, s=1 << 16):
    r = ctypes.c_int(0)
    return lib.sb_jacobi(g, s, ni, nj, nk, iters, 0.0, 1 / 6, depth, None, ctypes.byref(r))


def test_argument_errors_map_to_reference_exceptions():
    lib = _lib.load()
    with pytest.raises(DimensionError):
        _lib.check(_jac(lib, ni=0))
    with pytest.raises(PlanError):
        _lib.check(_jac(lib, iters=-1))
    with pytest.raises(PlanError):
        _lib.check(_jac(lib, depth=9))
    with pytest.raises(ValueError):
        _lib.check(_jac(lib, g=0))
    with pytest.raises(PlanError):
        _lib.check(lib.sb_gs(1 << 12, 4, 4, 4, 1, 0.1, 0, None))  # jacobi id on the GS entry
    lo, hi, gl, gh = (ctypes.c_int64() for _ in range(4))
    with pytest.raises(PartitionError):
        _lib.check(lib.sb_slab_layout(4, 5, 0, 1, *map(ctypes.byref, (lo, hi, gl, gh))))


def test_zero_iterations_is_a_no_op_without_device():
    lib = _lib.load()
    assert _jac(lib, iters=0) == 0
    assert lib.sb_gs(1 << 12, 4, 4, 4, 0, 0.1, 1, None) == 0


def test_slab_layout_matches_partition_blocks():
    from paper_1004_1741_b200.sweeps import partition_blocks

    lib = _lib.load()
    for nk, n, depth in [(10, 3, 2), (2048, 8, 4), (17, 4, 1), (9, 1, 8)]:
        ranges = partition_blocks(nk, n)
        for s in range(n):
            lo, hi, gl, gh = (ctypes.c_int64() for _ in range(4))
            _lib.check(lib.sb_slab_layout(nk, n, s, depth, *map(ctypes.byref, (lo, hi, gl, gh))))
            assert (lo.value - 1, hi.value - 1) == ranges[s]
            assert gl.value == (1 if s == 0 else depth)
            assert gh.value == (1 if s == n - 1 else depth)


# ---------------------------------------------------------------------------
# work schedule of the fused Jacobi launch (sb_jacobi_schedule, host only)

@pytest.mark.parametrize("sweeps,ni,nj,k_lo,k_hi,ctas", [
    (4, 1024, 1024, 1, 1025, 148),   # headline: whole-k bulk rounds + k-piece tail
    (3, 1024, 1024, 1, 1025, 148),
    (4, 512, 512, 1, 513, 148),
    (4, 128, 128, 1, 129, 148),      # fewer tiles than CTAs
    (4, 1024, 1024, 5, 1021, 148),   # a slab interior (sb_jacobi_planes)
    (4, 1024, 1024, 1, 5, 148),      # a slab edge
    (2, 1024, 1024, 1, 1025, 148),   # HBM-bound depths: regular k-blocks
    (1, 512, 256, 1, 300, 132),
    (8, 512, 512, 9, 505, 148),
    (4, 70, 1000, 1, 77, 7),
])
def test_schedule_covers_every_tile_plane_once(sweeps, ni, nj, k_lo, k_hi, ctas):
    import numpy as np

    items, (to, tj, ti_n, tj_n) = _lib.jacobi_schedule(sweeps, ni, nj, k_lo, k_hi, ctas)
    # the tiles cover the interior [1, ni] x [1, nj]
    assert to * ti_n >= ni + 1 and to * (ti_n - 1) < ni + 1
    assert tj * tj_n >= nj and tj * (tj_n - 1) < nj
    cover = np.zeros((tj_n, ti_n, k_hi - k_lo), dtype=np.int32)
    for ti, tjj, k0, k1 in items:
        assert 0 <= ti < ti_n and 0 <= tjj < tj_n and k_lo <= k0 < k1 <= k_hi
        cover[tjj, ti, k0 - k_lo:k1 - k_lo] += 1
    assert cover.min() == 1 and cover.max() == 1


def test_schedule_headline_uses_whole_k_border_first_list():
    import numpy as np

    items, (to, tj, ti_n, tj_n) = _lib.jacobi_schedule(4, 1024, 1024, 1, 1025, 148)
    assert (to, tj, ti_n, tj_n) == (56, 26, 19, 40)
    full = (items[:, 2] == 1) & (items[:, 3] == 1025)
    nbulk = (ti_n * tj_n // 148) * 148
    assert full[:nbulk].all() and not full[nbulk:].any()
    # border tiles (SEL steps) are claimed first
    border = (items[:, 0] == 0) | (items[:, 0] == ti_n - 1) | (items[:, 1] == 0) | \
             (items[:, 1] == tj_n - 1)
    nb = int(np.count_nonzero(border[:nbulk]))
    assert border[:nb].all()


def test_schedule_rejects_bad_arguments():
    lib = _lib.load()
    n = ctypes.c_int64(0)
    assert lib.sb_jacobi_schedule(9, 64, 64, 1, 9, 148, None, 0, ctypes.byref(n), None) != 0
    assert lib.sb_jacobi_schedule(4, 63, 64, 1, 9, 148, None, 0, ctypes.byref(n), None) != 0
    assert lib.sb_jacobi_schedule(4, 64, 64, 5, 5, 148, None, 0, ctypes.byref(n), None) != 0
    assert lib.sb_jacobi_schedule(4, 64, 64, 1, 9, 0, None, 0, ctypes.byref(n), None) != 0
    assert lib.sb_jacobi_schedule(4, 64, 64, 1, 9, 148, None, 0, ctypes.byref(n), None) == 0
    assert n.value > 0


def test_release_caches_without_device_is_a_no_op():
    lib = _lib.load()
    if _lib.device_count() == 0:
        assert lib.sb_release_caches(-1) == 0


def test_debug_fault_hook_validates_its_arguments():
    """sb_debug_fault (fault-injection test hook) needs no device; an unknown
    kind is an argument error, 0 restores normal operation."""
    lib = _lib.load()
    with pytest.raises(ValueError):
        _lib.check(lib.sb_debug_fault(7, 0))
    _lib.check(lib.sb_debug_fault(0, 0))
