"""Jacobi z-slabs on one GPU: sb_jacobi_slabs with G slabs of config 4's
1024^3 grid (all on GPU 0, one stream, so the slabs run one after another)
against sb_jacobi on the whole grid, 100 sweeps at depth 4.  The ratio is
the cost of the slab schedule itself -- ghost zones recomputed, the edge
launches that also write the neighbours' ghost planes (the fused exchange)
-- i.e. the compute side of multi-GPU weak scaling."""
import ctypes
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1004_1741_b200 import _lib  # noqa: E402
from paper_1004_1741_b200.slabs import slab_layout  # noqa: E402

n, sweeps, depth = 1024, 100, 4
lib = _lib.load()
st = torch.cuda.Stream()
sp = ctypes.c_void_p(st.cuda_stream)


def timed(fn, reps=2):
    fn()
    best = None
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fn()
        e1.record(st)
        torch.cuda.synchronize()
        sec = e0.elapsed_time(e1) / 1e3
        best = sec if best is None else min(best, sec)
    return best


whole = torch.rand((n + 2, n + 2, n + 2), dtype=torch.float64, device="cuda")
scratch = torch.empty_like(whole)
r = ctypes.c_int(0)
base = timed(lambda: _lib.check(lib.sb_jacobi(whole.data_ptr(), scratch.data_ptr(), n, n, n, sweeps,
                                             0.0, 1 / 6, depth, sp, ctypes.byref(r))))
print(json.dumps({"G": "sb_jacobi", "mlups": sweeps * n ** 3 / base / 1e6}), flush=True)
del scratch
for G in (2, 4):
    bufs, scr = [], []
    for s in range(G):
        own_lo, own_hi, glo, ghi = slab_layout(n, G, s, depth)
        bufs.append(whole[own_lo - glo:own_hi + ghi].clone())
        scr.append(torch.empty_like(bufs[-1]))
    devs = (ctypes.c_int * G)(*([0] * G))
    pa = (ctypes.c_void_p * G)(*[t.data_ptr() for t in bufs])
    ps = (ctypes.c_void_p * G)(*[t.data_ptr() for t in scr])
    pst = (ctypes.c_void_p * G)(*([st.cuda_stream] * G))
    sec = timed(lambda: _lib.check(lib.sb_jacobi_slabs(G, devs, pa, ps, n, n, n, sweeps, 0.0, 1 / 6,
                                                       depth, pst, ctypes.byref(r))))
    print(json.dumps({"G": G, "mlups": sweeps * n ** 3 / sec / 1e6, "vs_sb_jacobi": base / sec}),
          flush=True)
    del bufs, scr
