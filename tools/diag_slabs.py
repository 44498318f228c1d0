"""Dev: isolate z-slab issues: restricted-range blocks and 1-slab runs."""
import ctypes, sys
from pathlib import Path
R = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(R)); sys.path.insert(0, str(R / "oracle")); sys.path.insert(0, str(R / "tests"))
import numpy as np, torch, oracle
from conftest import make_input, sha
from paper_1004_1741_b200 import _lib
from paper_1004_1741_b200.slabs import slab_layout
lib = _lib.load()
g = make_input({"shape": [64, 30, 40], "pattern": "random", "seed": 9, "lo": 0.0, "hi": 1.0})
for T in (1, 2, 3):
    want = oracle.run_serial("jacobi", g.data, T, 0.0, 1/6)
    for (lo, hi) in [(1, 41), (1, 10), (10, 41), (5, 20), (20, 21)]:
        a = torch.from_numpy(g.data.copy()).cuda(); b = torch.from_numpy(g.data.copy()).cuda()
        _lib.check(lib.sb_jacobi_planes(a.data_ptr(), b.data_ptr(), 64, 30, 40, lo, hi, T, 0.0, 1/6, None)); torch.cuda.synchronize()
        got = b.cpu().numpy()
        ok = np.array_equal(got[lo:hi], want[lo:hi]); untouched = np.array_equal(np.delete(got, range(lo, hi), 0), np.delete(g.data, range(lo, hi), 0))
        print(f"planes T={T} [{lo},{hi}): out-ok={ok} rest-untouched={untouched}", flush=True)
for nslabs, depth, iters in [(1, 2, 7), (2, 2, 2), (2, 2, 4), (2, 2, 7), (2, 1, 3)]:
    want = oracle.run_serial("jacobi", g.data, iters, 0.0, 1/6)
    bufs, scr = [], []
    for s in range(nslabs):
        lo, hi, gl, gh = slab_layout(g.nk, nslabs, s, depth)
        part = torch.from_numpy(np.ascontiguousarray(g.data[lo - gl:hi + gh])).cuda(); bufs.append(part); scr.append(torch.empty_like(part))
    devs = (ctypes.c_int * nslabs)(*([0] * nslabs))
    pa = (ctypes.c_void_p * nslabs)(*[t.data_ptr() for t in bufs]); pb = (ctypes.c_void_p * nslabs)(*[t.data_ptr() for t in scr])
    streams = [torch.cuda.Stream() for _ in range(nslabs)]; ps = (ctypes.c_void_p * nslabs)(*[s.cuda_stream for s in streams])
    res = ctypes.c_int(-1)
    rc = lib.sb_jacobi_slabs(nslabs, devs, pa, pb, 64, 30, 40, iters, 0.0, 1/6, depth, ps, ctypes.byref(res))
    torch.cuda.synchronize()
    msgs = []
    for s in range(nslabs):
        lo, hi, gl, gh = slab_layout(g.nk, nslabs, s, depth)
        t = (scr if res.value else bufs)[s].cpu().numpy()[gl:gl + hi - lo]
        bad = np.argwhere(t != want[lo:hi])
        msgs.append(f"slab{s} bad={len(bad)} planes={sorted(set((bad[:,0]+lo).tolist()))[:8]}")
    print(f"slabs n={nslabs} depth={depth} iters={iters} rc={rc} res={res.value}: " + "; ".join(msgs), flush=True)
