import torch, time
n = 1 << 29  # 4 GiB of fp64
h1 = torch.empty(n, dtype=torch.float64).pin_memory()
h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d1 = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(h2d, d2h, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); t = time.perf_counter()
        if h2d:
            with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
        torch.cuda.synchronize(); best = min(best, time.perf_counter() - t)
    return best
gb = n * 8 / 1e9
t = run(1, 0); print(f"H2D alone {gb/t:.1f} GB/s")
t = run(0, 1); print(f"D2H alone {gb/t:.1f} GB/s")
t = run(1, 1); print(f"both concurrently {2*gb/t:.1f} GB/s aggregate")
import subprocess; print(subprocess.run(["nvidia-smi", "--query-gpu=pcie.link.gen.current,pcie.link.width.current", "--format=csv"], capture_output=True, text=True).stdout)
