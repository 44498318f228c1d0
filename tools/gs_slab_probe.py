"""Per-slab, per-sweep cost of the GS z-pipeline stages on one GPU (all
slabs on one stream, so they run one after another): projects what G GPUs
would sustain (one stage per GPU)."""
import ctypes
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1004_1741_b200 import _lib  # noqa: E402
from paper_1004_1741_b200.slabs import gs_slab_layout  # noqa: E402

n, sweeps = 512, 10
lib = _lib.load()
for G in (1, 2, 4, 8):
    bufs = []
    for s in range(G):
        lo, hi = gs_slab_layout(n, G, s)
        t = torch.rand((hi - lo + 2, n + 2, n + 2), dtype=torch.float64, device="cuda")
        bufs.append(t)
    st = torch.cuda.Stream()
    devs = (ctypes.c_int * G)(*([0] * G))
    pa = (ctypes.c_void_p * G)(*[t.data_ptr() for t in bufs])
    ps = (ctypes.c_void_p * G)(*([st.cuda_stream] * G))
    _lib.check(lib.sb_gs_slabs(G, devs, pa, n, n, n, 2, 1 / 6, 1, ps))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _lib.check(lib.sb_gs_slabs(G, devs, pa, n, n, n, sweeps, 1 / 6, 1, ps))
    sec = time.perf_counter() - t0
    per_stage = sec / sweeps / G
    print(json.dumps({"G": G, "stage_sweep_us": per_stage * 1e6,
                      "projected_mlups_G_gpus": n ** 3 / (per_stage * (sweeps + G - 1) / sweeps) / 1e6}))
