"""Kernel names, coefficients and cost table of the drop-in (reference
``stencilbench.kernels``, pkg/src/stencilbench/kernels.py:26-55).

The arithmetic itself lives in libsb200.so (csrc/jacobi_tb.cuh, csrc/gs.cu)
and reproduces the reference's fixed summation orders bit for bit:

* jacobi:          a*c + b*(((((W+E)+S)+N)+D)+U)        (kernels.py:125-134)
* gs-naive:        b*(((((W+E)+S)+N)+D)+U), in place    (kernels.py:154-163)
* gs-interleaved:  b*(W + ((((E+S)+N)+D)+U)), in place  (kernels.py:165-187)
"""

import math
from dataclasses import dataclass

JACOBI = "jacobi"
GS_NAIVE = "gs-naive"
GS_INTERLEAVED = "gs-interleaved"
KERNELS = (JACOBI, GS_NAIVE, GS_INTERLEAVED)

# (adds, muls) per cell update (kernels.py:31-32)
KERNEL_COSTS = {JACOBI: (6, 2), GS_NAIVE: (5, 1), GS_INTERLEAVED: (5, 1)}


@dataclass(frozen=True)
class StencilCoeffs:
    """Centre weight a (Jacobi only) and neighbour weight b; both finite."""

    a: float
    b: float

    def __post_init__(self):
        if not (math.isfinite(self.a) and math.isfinite(self.b)):
            raise ValueError(f"non-finite stencil coefficients ({self.a}, {self.b})")


# ---------------------------------------------------------------------------
# line-level operations (reference kernels.py:212-247), on the GPU

def _check_line(g, k, j):
    from .errors import BoundsError

    if not (0 <= k < g.nk and 0 <= j < g.nj):
        raise BoundsError(f"line (k={k}, j={j}) outside interior of {g.nk}x{g.nj} planes")


def _device_view(g):
    """(tensor on the GPU, write-back callable) for a host or device grid."""
    import torch

    if type(g.data).__module__.startswith("torch"):
        return g.data, lambda t: None
    t = torch.from_numpy(g.data).cuda()

    def back(tt):
        g.data[...] = tt.cpu().numpy()

    return t, back


def _line(kernel, src, dst, a, b, k, j):
    import ctypes

    import torch

    from . import _lib

    lib = _lib.load()
    _lib.require_device()
    s, s_back = _device_view(src)
    d, d_back = _device_view(dst) if dst is not None else (None, lambda t: None)
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    _lib.check(lib.sb_line_update(_lib.KERNEL_IDS[kernel], s.data_ptr(),
                                  d.data_ptr() if d is not None else None,
                                  src.ni, src.nj, src.nk, k, j, a, b, st))
    _lib.check(lib.sb_sync(st))
    if dst is not None:
        d_back(d)
    else:
        s_back(s)


def _shares_memory(x, y):
    if type(x).__module__.startswith("torch"):
        return x.data_ptr() == y.data_ptr() if type(y).__module__.startswith("torch") else False
    import numpy as np

    return (not type(y).__module__.startswith("torch")) and np.shares_memory(x, y)


def jacobi_line_update(src, dst, coeffs, k, j):
    """Out-of-place 7-point update of interior line (k, j): dst only written,
    src only read (reference kernels.py:220-233)."""
    from .errors import AliasingError, ShapeError

    if not src.same_extents(dst):
        raise ShapeError(f"src {src.ni}x{src.nj}x{src.nk} vs dst {dst.ni}x{dst.nj}x{dst.nk}")
    if _shares_memory(src.data, dst.data):
        raise AliasingError("jacobi_line_update requires distinct src/dst storage")
    _check_line(src, k, j)
    _line(JACOBI, src, dst, coeffs.a, coeffs.b, k, j)


def gs_line_update(g, b, k, j):
    """In-place lexicographic Gauss-Seidel update of interior line (k, j)."""
    _check_line(g, k, j)
    _line(GS_NAIVE, g, None, 0.0, b, k, j)


def gs_line_update_interleaved(g, b, k, j):
    """Same recurrence as gs_line_update with the interleaved association
    (differs by one reassociated addition per cell)."""
    _check_line(g, k, j)
    _line(GS_INTERLEAVED, g, None, 0.0, b, k, j)
