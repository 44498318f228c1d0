"""Dev: GS wait-time breakdown with the SB_GS_PROFILE build."""
import ctypes, sys
from pathlib import Path
import torch
lib = ctypes.CDLL(str(Path(__file__).resolve().parent / "libsb200_prof.so"))
lib.sb_gs.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_double, ctypes.c_int, ctypes.c_void_p]
lib.sb_gs_profile.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
for (n, nj, nk, it) in [(512, 512, 512, 20)]:
    g = torch.rand((nk + 2, nj + 2, n + 2), dtype=torch.float64, device="cuda")
    lib.sb_gs(g.data_ptr(), n, nj, nk, 1, 1/6, 1, None); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); rc = lib.sb_gs(g.data_ptr(), n, nj, nk, it, 1/6, 1, None); e1.record(); torch.cuda.synchronize()
    out = (ctypes.c_ulonglong * 6)(); lib.sb_gs_profile(out)
    tot, ws, wc, nt, le, ld = list(out)
    print(f"{n}x{nj}x{nk}x{it}: {e0.elapsed_time(e1):.3f} ms rc={rc}; per-CTA cycles total {tot/148:.3g}; "
          f"wait task-start {100*ws/tot:.1f}%, wait chunk {100*wc/tot:.1f}%, tasks {nt}; "
          f"loader: waiting for a free slot {100*le/tot:.2f}% ({le:.3g} cyc), for dependencies {100*ld/tot:.2f}% ({ld:.3g})", flush=True)
