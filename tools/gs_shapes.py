"""Dev: GS timing across shapes to separate per-step cost from inter-tile lag."""
import ctypes, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_1004_1741_b200 import _lib
lib = _lib.load()
st = torch.cuda.current_stream(); sp = ctypes.c_void_p(st.cuda_stream)
for (ni, nj, nk, it) in [(512,16,16,1),(512,16,16,4),(512,32,32,1),(512,512,16,1),(512,16,512,1),(512,64,64,1),(512,128,128,1),(512,512,512,1),(512,512,512,4),(512,512,512,16),(1024,256,256,4)]:
    g = torch.rand((nk+2, nj+2, ni+2), dtype=torch.float64, device="cuda")
    _lib.check(lib.sb_gs(g.data_ptr(), ni, nj, nk, 1, 1/6, 1, sp)); _lib.check(lib.sb_sync(sp))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st); _lib.check(lib.sb_gs(g.data_ptr(), ni, nj, nk, it, 1/6, 1, sp)); e1.record(st); _lib.check(lib.sb_sync(sp))
    ms = e0.elapsed_time(e1)
    tiles = ((nj+15)//16)*((nk+15)//16)
    print(f"{ni}x{nj}x{nk} sweeps={it} tiles={tiles}: {ms:.3f} ms, {it*ni*nj*nk/ms/1e3:.0f} MLUP/s, us/step(1 tile path)={ms*1e3/((ni+30)*it):.3f}", flush=True)
