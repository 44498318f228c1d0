"""Dev: locate Jacobi mismatches vs the oracle for a shape over depths/iters."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent)); sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "oracle"))
import numpy as np, torch, oracle
from paper_1004_1741_b200 import InitPattern, create_grid
from paper_1004_1741_b200.grid import Grid3D
from paper_1004_1741_b200.sweeps import execute
ni, nj, nk = (int(x) for x in sys.argv[1].split("x"))
a = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
host = create_grid(ni, nj, nk, InitPattern.seeded_random(42))
for depth in (1, 2, 3, 4):
    for iters in (depth, 2 * depth, 11):
        want = oracle.run_serial("jacobi", host.data, iters, a, 1 / 6)
        g = Grid3D(ni, nj, nk, torch.from_numpy(host.data.copy()).cuda())
        execute("jacobi", g, iters, a, 1 / 6, depth)
        got = g.data.cpu().numpy()
        bad = np.argwhere(got != want)
        msg = "ok" if len(bad) == 0 else f"{len(bad)} bad; first {bad[:4].tolist()} last {bad[-2:].tolist()} kset {sorted(set(bad[:,0].tolist()))[:12]} jset {sorted(set(bad[:,1].tolist()))[:12]} iset {sorted(set(bad[:,2].tolist()))[:12]}"
        print(f"{ni}x{nj}x{nk} depth {depth} iters {iters}: {msg}", flush=True)
