"""Dev probe: time the hot-path kernels on one GPU with CUDA events.

    python tools/probe.py [--n 512] [--iters 8] [--depths 1,2,4,8] [--gs]
"""

import argparse
import ctypes
import json
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_1004_1741_b200 import _lib  # noqa: E402

PEAK = 6534.5e9


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--iters", type=int, default=8)
    ap.add_argument("--depths", default="1,2,4,8")
    ap.add_argument("--gs", action="store_true")
    ap.add_argument("--gs-iters", type=int, default=4)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    lib = _lib.load()
    n = args.n
    g = torch.rand((n + 2, n + 2, n + 2), dtype=torch.float64, device="cuda")
    s = torch.empty_like(g)
    st = torch.cuda.current_stream()
    sp = ctypes.c_void_p(st.cuda_stream)
    cells = n ** 3
    res = {}
    for d in [int(x) for x in args.depths.split(",") if x and x != "none"]:
        in_s = ctypes.c_int(0)
        iters = max(d, (args.iters // d) * d)
        _lib.check(lib.sb_jacobi(g.data_ptr(), s.data_ptr(), n, n, n, iters, 0.0, 1 / 6, d, sp,
                                 ctypes.byref(in_s)))
        _lib.check(lib.sb_sync(sp))
        best = 1e9
        for _ in range(args.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            _lib.check(lib.sb_jacobi(g.data_ptr(), s.data_ptr(), n, n, n, iters, 0.0, 1 / 6, d, sp,
                                     ctypes.byref(in_s)))
            e1.record(st)
            _lib.check(lib.sb_sync(sp))
            best = min(best, e0.elapsed_time(e1) / 1e3)
        mlups = iters * cells / best / 1e6
        res[f"jacobi_T{d}"] = {"ms": best * 1e3, "mlups": mlups,
                               "hbm_frac_algo": mlups * 1e6 * 16 / d / PEAK,
                               "roof1_frac": mlups * 1e6 * 16 / PEAK}
        print(json.dumps({f"jacobi_T{d}": res[f"jacobi_T{d}"]}), flush=True)
    if args.gs:
        for kid, name in ((1, "gs-naive"), (2, "gs-interleaved")):
            iters = args.gs_iters
            _lib.check(lib.sb_gs(g.data_ptr(), n, n, n, 1, 1 / 6, kid, sp))
            _lib.check(lib.sb_sync(sp))
            t0 = time.perf_counter()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            _lib.check(lib.sb_gs(g.data_ptr(), n, n, n, iters, 1 / 6, kid, sp))
            e1.record(st)
            _lib.check(lib.sb_sync(sp))
            sec = e0.elapsed_time(e1) / 1e3
            mlups = iters * cells / sec / 1e6
            print(json.dumps({name: {"ms": sec * 1e3, "mlups": mlups,
                                     "roof1_frac": mlups * 1e6 * 16 / PEAK,
                                     "wall": time.perf_counter() - t0}}), flush=True)


if __name__ == "__main__":
    main()
