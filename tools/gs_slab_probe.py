"""GS z-pipeline on one GPU: sb_gs_slabs with G slabs (all on GPU 0, one
fused launch: the slabs' edge-plane chunks are pushed into the neighbours'
ghost planes exactly as between GPUs) against sb_gs on the whole grid, at
config 5's size (512^3, 100 sweeps).  The ratio is the cost of the slab
protocol itself (ghost flags, pushes, partial tiles at the seams)."""
import ctypes
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1004_1741_b200 import _lib  # noqa: E402
from paper_1004_1741_b200.slabs import gs_slab_layout  # noqa: E402

n, sweeps = 512, 100
lib = _lib.load()
whole = torch.rand((n + 2, n + 2, n + 2), dtype=torch.float64, device="cuda") * 2 - 1
st = torch.cuda.Stream()


def timed(fn, reps=3):
    best = None
    fn()  # warm-up
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)
        fn()
        e1.record(st)
        torch.cuda.synchronize()
        sec = e0.elapsed_time(e1) / 1e3
        best = sec if best is None else min(best, sec)
    return best


sp = ctypes.c_void_p(st.cuda_stream)
base = timed(lambda: _lib.check(lib.sb_gs(whole.data_ptr(), n, n, n, sweeps, 1 / 6, 1, sp)))
print(json.dumps({"G": "sb_gs", "mlups": sweeps * n ** 3 / base / 1e6}), flush=True)
for G in (2, 4, 8):
    bufs = []
    for s in range(G):
        lo, hi = gs_slab_layout(n, G, s)
        bufs.append(whole[lo - 1:hi + 1].clone())
    devs = (ctypes.c_int * G)(*([0] * G))
    pa = (ctypes.c_void_p * G)(*[t.data_ptr() for t in bufs])
    ps = (ctypes.c_void_p * G)(*([st.cuda_stream] * G))
    sec = timed(lambda: _lib.check(lib.sb_gs_slabs(G, devs, pa, n, n, n, sweeps, 1 / 6, 1, ps)))
    print(json.dumps({"G": G, "mlups": sweeps * n ** 3 / sec / 1e6, "vs_sb_gs": base / sec}), flush=True)
