"""The reference-side binding shown in INTEGRATION.md section 2 runs as
written against the built library: its error mapping and early returns work
without a GPU (every check it relies on happens before any device work)."""

import re
import types
from pathlib import Path

import numpy as np
import pytest

from paper_1004_1741_b200 import _lib

ROOT = Path(__file__).resolve().parent.parent


class StencilError(Exception):
    pass


class DimensionError(StencilError):
    pass


class PlanError(StencilError):
    pass


class PartitionError(StencilError):
    pass


class ConfigError(StencilError):
    pass


@pytest.fixture(scope="module")
def binding():
    text = (ROOT / "INTEGRATION.md").read_text()
    sec = text[text.index("## 2. Reference-side binding"):]
    code = re.search(r"```python\n(.*?)```", sec, flags=re.S).group(1)
    code = code.replace("from ..errors import DimensionError, PlanError, PartitionError, "
                        "ConfigError, StencilError\n", "")
    code = code.replace('"/path/to/libsb200.so"', repr(str(_lib.LIB_PATH)))
    ns = {"DimensionError": DimensionError, "PlanError": PlanError,
          "PartitionError": PartitionError, "ConfigError": ConfigError,
          "StencilError": StencilError}
    exec(compile(code, "INTEGRATION.md", "exec"), ns)  # noqa: S102
    return ns["run_b200"]


def _plan(kernel="jacobi", iters=3, variant="serial", t=2):
    return types.SimpleNamespace(kernel=kernel, iter_end=iters, variant=variant,
                                 coeffs=types.SimpleNamespace(a=0.0, b=1 / 6),
                                 config=types.SimpleNamespace(threads_per_group=t))


def _grid(ni, nj, nk):
    return types.SimpleNamespace(ni=ni, nj=nj, nk=nk,
                                 data=np.zeros((nk + 2, nj + 2, ni + 2), dtype=np.float64))


def test_zero_iterations_return_the_grid(binding):
    g = _grid(4, 4, 4)
    assert binding(_plan(iters=0), g) is g


def test_errors_map_to_reference_exceptions(binding):
    with pytest.raises(DimensionError):
        binding(_plan(), _grid(0, 4, 4))
    with pytest.raises(PlanError):
        binding(_plan(iters=-1), _grid(4, 4, 4))



def test_no_device_is_an_error_not_a_fallback(binding):
    """A valid plan without a GPU fails loudly (no CPU fallback)."""
    if _lib.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(StencilError):
        binding(_plan(variant="wavefront", t=4), _grid(8, 6, 5))


@pytest.fixture(scope="module")
def multi_binding(binding):
    """INTEGRATION.md section 4's run_b200_multi, executed on top of the
    section 2 namespace (it reuses _lib, _KID and _EXC)."""
    text = (ROOT / "INTEGRATION.md").read_text()
    sec = text[text.index("## 2. Reference-side binding"):]
    code2 = re.search(r"```python\n(.*?)```", sec, flags=re.S).group(1)
    code2 = code2.replace("from ..errors import DimensionError, PlanError, PartitionError, "
                          "ConfigError, StencilError\n", "")
    code2 = code2.replace('"/path/to/libsb200.so"', repr(str(_lib.LIB_PATH)))
    sec4 = text[text.index("## 4. Multi-GPU"):]
    code4 = re.search(r"```python\n(.*?)```", sec4, flags=re.S).group(1)
    ns = {"DimensionError": DimensionError, "PlanError": PlanError,
          "PartitionError": PartitionError, "ConfigError": ConfigError,
          "StencilError": StencilError}
    exec(compile(code2 + "\n" + code4, "INTEGRATION.md", "exec"), ns)  # noqa: S102
    return ns["run_b200_multi"]


def test_multi_binding_errors_before_any_work(multi_binding):
    g = _grid(4, 4, 3)
    assert multi_binding(_plan(iters=0), g, [0, 0]) is g
    with pytest.raises(PartitionError):  # more GPUs than planes
        multi_binding(_plan(), g, [0, 0, 0, 0])
    with pytest.raises(DimensionError):
        multi_binding(_plan(), _grid(0, 4, 4), [0])
    with pytest.raises(PlanError):
        multi_binding(_plan(iters=-2), g, [0])
