"""ctypes binding of libsb200.so (C ABI: include/stencil_b200.h).

The shared library is the product: there is no CPU fallback.  Loading fails
loudly (DeviceError) when the library is missing; device calls fail loudly
when no CUDA device is visible.
"""

import ctypes
import os
from pathlib import Path

import numpy as np

from .errors import (
    ConfigError,
    DeviceError,
    DimensionError,
    PartitionError,
    PlanError,
)

# SB200_LIB: load an alternative build (experiments); default: the in-tree library
LIB_PATH = Path(os.environ.get("SB200_LIB") or Path(__file__).resolve().parent / "libsb200.so")

SB_OK = 0
KERNEL_IDS = {"jacobi": 0, "gs-naive": 1, "gs-interleaved": 2}

_i64 = ctypes.c_int64
_dbl = ctypes.c_double
_int = ctypes.c_int
_vp = ctypes.c_void_p
_pd = ctypes.POINTER(ctypes.c_double)

# name -> (restype, argtypes); every symbol declared in include/stencil_b200.h
SIGNATURES = {
    "sb_version": (_int, []),
    "sb_last_error": (ctypes.c_char_p, []),
    "sb_device_count": (_int, []),
    "sb_max_depth": (_int, []),
    "sb_jacobi_schedule": (_int, [_int, _i64, _i64, _i64, _i64, _int,
                                  ctypes.POINTER(ctypes.c_int32), _i64, ctypes.POINTER(_i64),
                                  ctypes.POINTER(ctypes.c_int32)]),
    "sb_jacobi": (_int, [_vp, _vp, _i64, _i64, _i64, _i64, _dbl, _dbl, _int, _vp,
                         ctypes.POINTER(_int)]),
    "sb_gs": (_int, [_vp, _i64, _i64, _i64, _i64, _dbl, _int, _vp]),
    "sb_sync": (_int, [_vp]),
    "sb_debug_fault": (_int, [_int, _i64]),
    "sb_line_update": (_int, [_int, _vp, _vp, _i64, _i64, _i64, _i64, _i64, _dbl, _dbl, _vp]),
    "sb_reference_sweeps": (_int, [_int, _vp, _vp, _i64, _i64, _i64, _i64, _dbl, _dbl, _vp,
                                   ctypes.POINTER(_int)]),
    "sb_run_host": (_int, [_int, _vp, _i64, _i64, _i64, _i64, _dbl, _dbl, _int, _int]),
    "sb_run_host_batch": (_int, [_int, _vp, _int, _i64, _i64, _i64, _i64, _dbl, _dbl, _int, _int]),
    "sb_triad": (_int, [_vp, _vp, _vp, _dbl, _i64, _vp]),
    "sb_fp64_probe": (_int, [_vp, _i64, _vp, ctypes.POINTER(_i64)]),
    "sb_host_alloc": (_vp, [_i64]),
    "sb_release_caches": (_int, [_int]),
    "sb_host_free": (None, [_vp]),
    "sb_jacobi_planes": (_int, [_vp, _vp, _i64, _i64, _i64, _i64, _i64, _int, _dbl, _dbl, _vp]),
    "sb_slab_layout": (_int, [_i64, _int, _int, _int, ctypes.POINTER(_i64), ctypes.POINTER(_i64),
                              ctypes.POINTER(_i64), ctypes.POINTER(_i64)]),
    "sb_jacobi_slabs": (_int, [_int, ctypes.POINTER(_int), ctypes.POINTER(_vp), ctypes.POINTER(_vp),
                               _i64, _i64, _i64, _i64, _dbl, _dbl, _int, ctypes.POINTER(_vp),
                               ctypes.POINTER(_int)]),
    "sb_gs_slab_layout": (_int, [_i64, _int, _int, ctypes.POINTER(_i64), ctypes.POINTER(_i64)]),
    "sb_gs_slabs": (_int, [_int, ctypes.POINTER(_int), ctypes.POINTER(_vp), _i64, _i64, _i64, _i64,
                           _dbl, _int, ctypes.POINTER(_vp)]),
    "sb_run_multi": (_int, [_int, _vp, _i64, _i64, _i64, _i64, _dbl, _dbl, _int, _int,
                            ctypes.POINTER(_int)]),
}

_lib = None


def load():
    """Load libsb200.so once; raise DeviceError if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise DeviceError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "or `make -C paper_1004_1741_b200/csrc` (no CPU fallback exists)"
        )
    # let libcudart resolve to the copy torch already loaded, when present
    try:
        import torch  # noqa: F401
    except ImportError:
        pass
    lib = ctypes.CDLL(str(LIB_PATH), mode=os.RTLD_LOCAL | getattr(os, "RTLD_NOW", 2))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


_ERRORS = {
    1: DimensionError,
    2: PlanError,
    3: ConfigError,
    4: PartitionError,
    5: DeviceError,
    6: DeviceError,
    7: ValueError,
    8: DeviceError,
}


def check(status):
    """Map an sb_status to the reference's exception classes."""
    if status == SB_OK:
        return
    msg = load().sb_last_error().decode(errors="replace")
    raise _ERRORS.get(status, DeviceError)(msg or f"libsb200 status {status}")


def device_count():
    return load().sb_device_count()


def require_device():
    if device_count() < 1:
        raise DeviceError("no CUDA device visible: the B200 engines have no CPU fallback")


def max_depth():
    return load().sb_max_depth()


def release_caches(device=-1):
    """Free the device buffers cached between host-entry calls
    (sb_release_caches)."""
    check(load().sb_release_caches(device))


def jacobi_schedule(sweeps, ni, nj, k_lo, k_hi, ctas):
    """Work items of one fused Jacobi launch (sb_jacobi_schedule; host only):
    returns (items, (TO, TJ, tiles_i, tiles_j)) with items an (n, 4) int32
    array of (tile_i, tile_j, k0, k1) in claim order."""
    import numpy as np

    lib = load()
    n = _i64(0)
    dims = (ctypes.c_int32 * 4)()
    check(lib.sb_jacobi_schedule(sweeps, ni, nj, k_lo, k_hi, ctas, None, 0, ctypes.byref(n), dims))
    items = np.zeros((max(1, n.value), 4), dtype=np.int32)
    check(lib.sb_jacobi_schedule(sweeps, ni, nj, k_lo, k_hi, ctas,
                                 items.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), n.value,
                                 ctypes.byref(n), dims))
    return items[:n.value], tuple(dims)


def pinned_array(shape):
    """Page-locked float64 host array (freed when the array is collected)."""
    count = int(np.prod(shape))
    lib = load()
    ptr = lib.sb_host_alloc(count)
    if not ptr:
        raise MemoryError(lib.sb_last_error().decode(errors="replace"))
    buf = (ctypes.c_double * count).from_address(ptr)
    arr = np.frombuffer(buf, dtype=np.float64).reshape(shape)
    # keep the allocation alive as long as the array; free on collection
    holder = _PinnedHolder(ptr)
    arr_base = np.ndarray(shape, dtype=np.float64, buffer=arr.data)
    _pinned_owners[id(arr_base)] = holder
    import weakref

    weakref.finalize(arr_base, _release_pinned, id(arr_base))
    return arr_base


class _PinnedHolder:
    def __init__(self, ptr):
        self.ptr = ptr


_pinned_owners = {}


def _release_pinned(key):
    h = _pinned_owners.pop(key, None)
    if h is not None and _lib is not None:
        _lib.sb_host_free(h.ptr)
