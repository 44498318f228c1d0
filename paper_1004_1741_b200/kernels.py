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
