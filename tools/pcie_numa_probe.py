"""Does host-side placement change the PCIe duplex rate?  Prints the host's
NUMA layout, the GPU's local CPU list, and H2D / D2H / both-at-once rates
with the process (a) unpinned, (b) pinned to the GPU's local CPUs before the
pinned buffers are allocated and touched, (c) with copies cut into chunks."""
import os, subprocess, sys, time
import torch

def sh(cmd):
    try:
        return subprocess.run(cmd, shell=True, capture_output=True, text=True, timeout=20).stdout.strip()
    except Exception as e:  # noqa: BLE001
        return f"<{e}>"

print(sh("lscpu | grep -E 'Model name|Socket|NUMA|^CPU\\(s\\)'"))
print(sh("nvidia-smi topo -m | head -8"))
bus = sh("nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader -i 0").lower()
bus = bus[4:] if bus.startswith("0000") and len(bus) > 12 else bus
path = f"/sys/bus/pci/devices/{bus}"
print("gpu", bus, "numa_node", sh(f"cat {path}/numa_node"), "local_cpulist", sh(f"cat {path}/local_cpulist"))
print("affinity now:", sorted(os.sched_getaffinity(0)))

def parse(cl):
    out = set()
    for part in cl.split(","):
        if "-" in part:
            a, b = part.split("-"); out |= set(range(int(a), int(b) + 1))
        elif part.strip().isdigit():
            out.add(int(part))
    return out

def measure(tag, chunk=None):
    n = 1 << 29
    h1 = torch.empty(n, dtype=torch.float64).pin_memory(); h1.zero_()
    h2 = torch.empty(n, dtype=torch.float64).pin_memory(); h2.zero_()
    d1 = torch.empty(n, dtype=torch.float64, device="cuda"); d2 = torch.zeros(n, dtype=torch.float64, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    def copy(dst, src, st):
        with torch.cuda.stream(st):
            if chunk is None: dst.copy_(src, non_blocking=True)
            else:
                for o in range(0, n, chunk): dst[o:o + chunk].copy_(src[o:o + chunk], non_blocking=True)
    def run(a, b):
        best = 1e9
        for _ in range(3):
            torch.cuda.synchronize(); t = time.perf_counter()
            if a: copy(d1, h1, s1)
            if b: copy(h2, d2, s2)
            torch.cuda.synchronize(); best = min(best, time.perf_counter() - t)
        return best
    gb = n * 8 / 1e9
    print(f"{tag}: H2D {gb/run(1,0):.1f}  D2H {gb/run(0,1):.1f}  both {2*gb/run(1,1):.1f} GB/s", flush=True)

measure("unpinned process")
measure("unpinned, 64 MiB chunks", chunk=1 << 23)
local = parse(sh(f"cat {path}/local_cpulist"))
if local and local != os.sched_getaffinity(0):
    try:
        os.sched_setaffinity(0, local & os.sched_getaffinity(0) or local)
        print("affinity ->", sorted(os.sched_getaffinity(0)))
        measure("pinned to the GPU's CPUs")
    except OSError as e:
        print("setaffinity failed", e)
else:
    print("GPU-local CPU list equals the current affinity (or unknown): nothing to pin")
