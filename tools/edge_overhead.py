"""Per-GPU compute overhead of the z-slab schedule (an inner rank computes
its two 4-plane edges first, then the interior, every 4-sweep period) versus
one fused launch per period, on one GPU at 1024^3: the compute part of the
weak-scaling efficiency (the halo exchange itself runs concurrently)."""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1004_1741_b200 import _lib  # noqa: E402

n, d, periods = 1024, 4, 25
lib = _lib.load()
g = torch.rand((n + 2, n + 2, n + 2), dtype=torch.float64, device="cuda")
s = g.clone()
sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def run(split):
    bufs = (g, s)
    for p in range(periods):
        src, dst = bufs[p % 2], bufs[(p + 1) % 2]
        ranges = [(1, 1 + d), (n + 1 - d, n + 1), (1 + d, n + 1 - d)] if split else [(1, n + 1)]
        for lo, hi in ranges:
            _lib.check(lib.sb_jacobi_planes(src.data_ptr(), dst.data_ptr(), n, n, n, lo, hi, d,
                                            0.0, 1 / 6, sp))


for split in (False, True, False, True):
    run(split)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run(split)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{'edges+interior' if split else 'one launch'}: {ms:.2f} ms for {periods * d} sweeps, "
          f"{periods * d * n ** 3 / ms / 1e6:.0f} GLUP/s")
