"""Dev: run one small Jacobi launch (T from argv) and report the CUDA status."""
import ctypes, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_1004_1741_b200 import _lib
T = int(sys.argv[1]); n = int(sys.argv[2]) if len(sys.argv) > 2 else 48
lib = _lib.load()
g = torch.rand((n + 2, n + 2, n + 2), dtype=torch.float64, device="cuda")
s = torch.empty_like(g)
r = ctypes.c_int(0)
rc = lib.sb_jacobi(g.data_ptr(), s.data_ptr(), n, n, n, T, 0.0, 1 / 6, T, None, ctypes.byref(r))
print("launch rc", rc, lib.sb_last_error())
print("sync rc", lib.sb_sync(None), lib.sb_last_error())
