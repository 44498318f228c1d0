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
