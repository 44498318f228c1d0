"""Timing methodology, bandwidth probe and the bandwidth-ceiling model
(the drop-in's counterpart of the reference's ``stencilbench.perf``,
pkg/src/stencilbench/perf.py).

Model: with memory saturated a lattice-site update (LUP)
moves at least one 8-byte load and one 8-byte store, so

    P0 = M_S / bytes_per_lup        [LUP/s]

with M_S the sustained bandwidth (here measured on the GPU by
``stream_triad``).  Temporal blocking with depth t touches memory once per t
sweeps, so its traffic is the plain value divided by t.

``device="b200"`` gives the GPU's traffic: the Jacobi store stream is written
as whole L2 sectors (no write-allocate read), so plain Jacobi is 16 B/LUP, not
the 24 of a write-allocate CPU.  Without ``device`` the functions keep the
reference's CPU semantics exactly (its model tests are restated in
tests/test_perf.py).
"""

import ctypes
import math
import os
import platform
import sys
from dataclasses import dataclass, field
from datetime import datetime, timezone
from fractions import Fraction
from statistics import median

from .errors import ConfigError, DomainError
from .kernels import GS_INTERLEAVED, GS_NAIVE, JACOBI

STREAM_BYTES = 24  # triad a[i] = b[i] + s*c[i]: read b, read c, write a (full-sector stores)


def predict_p0(ms, bytes_per_lup):
    """Bandwidth-limited ceiling in LUP/s: exact quotient M_S / bytes
    (reference perf.py:86-92)."""
    if not (ms > 0 and bytes_per_lup > 0):
        raise DomainError(f"predict_p0 needs positive inputs, got ({ms}, {bytes_per_lup})")
    return ms / bytes_per_lup


_PLAIN = ("plain", "serial", "threaded", "pipeline")


def predict_traffic(kernel, variant, t=1, nt_stores=None, device=None):
    """Main-memory bytes per LUP as an exact Fraction (reference
    perf.py:98-119).  device="b200": GPU traffic (16 B/LUP for every plain
    sweep; ``nt_stores`` is meaningless there and must not be set)."""
    if t < 1:
        raise DomainError(f"blocking factor must be >= 1, got {t}")
    if kernel in (GS_NAIVE, GS_INTERLEAVED, "gs"):
        if nt_stores:
            raise DomainError("non-temporal stores are inapplicable to in-place GS")
        plain = Fraction(16)
    elif kernel == JACOBI:
        if device is not None:
            if nt_stores:
                raise DomainError("nt_stores has no meaning for the GPU model")
            plain = Fraction(16)
        else:
            plain = Fraction(16) if nt_stores else Fraction(24)
    else:
        raise DomainError(f"unknown kernel {kernel!r}")
    if variant in _PLAIN:
        return plain
    if variant == "wavefront":
        return plain / t
    raise DomainError(f"unknown variant {variant!r}")


def host_fingerprint(device=None):
    """Host + GPU description attached to every measurement record."""
    info = {
        "hostname": platform.node(),
        "machine": platform.machine(),
        "platform": platform.platform(),
        "python": sys.version.split()[0],
        "cpu_count": os.cpu_count(),
        "timestamp": datetime.now(timezone.utc).isoformat(timespec="seconds"),
    }
    try:
        import torch

        if torch.cuda.is_available():
            d = torch.cuda.current_device() if device is None else device
            p = torch.cuda.get_device_properties(d)
            info.update(gpu=p.name, gpu_sms=p.multi_processor_count,
                        gpu_mem_bytes=p.total_memory, torch=torch.__version__)
    except ImportError:
        pass
    return info


@dataclass
class StreamResult:
    bandwidth_bytes_per_s: float
    elements: int
    bytes_per_element: int
    seconds: list
    kernel: str
    validated: bool
    device: int = 0

    def to_dict(self):
        return dict(self.__dict__)


def stream_triad(elements=1 << 28, repetitions=5, warmup=1, device=0):
    """Sustained device bandwidth of a[i] = b[i] + s*c[i] (the reference's
    probe, perf.py:139-211, on the GPU): libsb200's sb_triad, CUDA-event
    timed, median of `repetitions`; validated on a sample like the reference."""
    import torch

    from . import _lib

    if elements <= 0:
        raise ConfigError(f"need a positive element count, got {elements}")
    _lib.require_device()
    lib = _lib.load()
    dev = torch.device("cuda", device)
    s = 3.0
    a = torch.zeros(elements, dtype=torch.float64, device=dev)
    b = torch.full((elements,), 1.5, dtype=torch.float64, device=dev)
    c = torch.full((elements,), 0.25, dtype=torch.float64, device=dev)
    idx = torch.randint(0, elements, (min(elements, 4),), generator=torch.Generator().manual_seed(7))
    b[idx] = torch.rand(len(idx), dtype=torch.float64).to(dev)
    c[idx] = torch.rand(len(idx), dtype=torch.float64).to(dev)
    with torch.cuda.device(dev):
        st = torch.cuda.current_stream()
        sp = ctypes.c_void_p(st.cuda_stream)
        seconds = []
        for rep in range(warmup + repetitions):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            _lib.check(lib.sb_triad(a.data_ptr(), b.data_ptr(), c.data_ptr(), s, elements, sp))
            e1.record(st)
            _lib.check(lib.sb_sync(sp))
            if rep >= warmup:
                seconds.append(e0.elapsed_time(e1) / 1e3)
    stride = max(1, elements // 4096)
    sample = slice(0, elements, stride)
    validated = bool(torch.equal(a[sample], b[sample] + s * c[sample]))
    if not validated:
        raise ArithmeticError("stream_triad validation failed: a != b + s*c")
    best = median(seconds)
    return StreamResult(bandwidth_bytes_per_s=elements * STREAM_BYTES / best, elements=elements,
                        bytes_per_element=STREAM_BYTES, seconds=seconds, kernel="sb_triad",
                        validated=validated, device=device)


def fp64_peak(iters=1 << 16, repetitions=3, device=0):
    """Sustained FP64 operation rate of the device (sb_fp64_probe:
    independent DADD chains on every SM, CUDA-event timed, best of
    `repetitions`), in DP operations per second -- the compute ceiling the
    stencil kernels are measured against besides HBM bandwidth."""
    import torch

    from . import _lib

    _lib.require_device()
    lib = _lib.load()
    dev = torch.device("cuda", device)
    sink = torch.zeros(256, dtype=torch.float64, device=dev)
    ops = ctypes.c_int64(0)
    best = None
    with torch.cuda.device(dev):
        st = torch.cuda.current_stream()
        sp = ctypes.c_void_p(st.cuda_stream)
        _lib.check(lib.sb_fp64_probe(sink.data_ptr(), 256, sp, ctypes.byref(ops)))  # warm-up
        for _ in range(repetitions):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            _lib.check(lib.sb_fp64_probe(sink.data_ptr(), iters, sp, ctypes.byref(ops)))
            e1.record(st)
            _lib.check(lib.sb_sync(sp))
            sec = e0.elapsed_time(e1) / 1e3
            best = sec if best is None else min(best, sec)
    return ops.value / best


@dataclass
class Measurement:
    kernel: str
    variant: str
    iter_end: int
    ni: int
    nj: int
    nk: int
    seconds: list
    repetitions: int
    warmup: int
    mlups: float  # from the median repetition
    depth: int = 1
    config: dict = field(default_factory=dict)
    flags: list = field(default_factory=list)
    host: dict = field(default_factory=dict)

    @property
    def median_seconds(self):
        return median(self.seconds)

    def to_dict(self):
        d = dict(self.__dict__)
        d["median_seconds"] = self.median_seconds
        return d


def measure(plan, grid_factory, repetitions=5, warmup=1, device="cuda", devices=None):
    """Run `plan` on identical fresh inputs (reference perf.py:241-297):
    `warmup` untimed runs, then `repetitions` timed ones.  Each input is
    created and moved to `device` outside the timed region; the timed region
    is the sweep call on the resident grid, bracketed by CUDA events on the
    current stream.  MLUP/s from the median.  With several `devices` (the
    threaded engines' z-slabs across GPUs) the call is synchronous over all
    of them and is timed by the host clock, slab scatter/gather included."""
    import time

    import torch

    from .sweeps import resolve_depth, run
    from .sweeps.engine import resolve_devices

    devs = resolve_devices(devices)
    multi = devs is not None and len(devs) > 1

    if repetitions < 1:
        raise ConfigError(f"need at least one repetition, got {repetitions}")
    seconds = []
    depth = 1
    g = None
    for rep in range(warmup + repetitions):
        g = grid_factory().to_device(device)
        depth = resolve_depth(plan, g)
        torch.cuda.synchronize()
        st = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(st)
        run(plan, g, devices=devs)
        e1.record(st)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        if rep >= warmup:
            seconds.append((t1 - t0) if multi else e0.elapsed_time(e1) / 1e3)
    med = median(seconds)
    total = plan.iter_end * g.ni * g.nj * g.nk
    cfg = {"threads": plan.threads, "gpus": len(devs) if multi else 1}
    if plan.config is not None:
        cfg.update(num_groups=plan.config.num_groups,
                   threads_per_group=plan.config.threads_per_group,
                   blocks=plan.config.blocks, barrier=plan.config.barrier)
    return Measurement(kernel=plan.kernel, variant=plan.variant, iter_end=plan.iter_end, ni=g.ni,
                       nj=g.nj, nk=g.nk, seconds=seconds, repetitions=repetitions, warmup=warmup,
                       mlups=(total / med / 1e6) if med > 0 else math.inf, depth=depth, config=cfg,
                       host=host_fingerprint())

