"""GS z-pipeline throughput at N GPUs (config 5: 512^3 x 100 sweeps,
U[-1,1), strong scaling), one process per GPU:

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \\
        tools/gs_multi_bench.py [--n 512] [--sweeps 100] [--kernel gs-naive]

Prints one JSON line (rank 0): MLUP/s of the whole job, timed on the device
as the max over ranks.  Not part of bench.py's contract (its multi-GPU
headline is the Jacobi weak-scaling config); correctness of the pipeline is
pinned by tests/test_slabs.py."""

import argparse
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    import torch.distributed as dist

    from paper_1004_1741_b200.slabs import GsSlabEngine, gpu_gs_compute

    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--sweeps", type=int, default=100)
    ap.add_argument("--kernel", default="gs-naive")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", 1))
    rank = int(os.environ.get("RANK", 0))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    n = args.n
    eng = GsSlabEngine(n, n, n, rank, world, gpu_gs_compute(n, n, 1 / 6, args.kernel),
                       like=torch.empty(0, dtype=torch.float64, device=dev))
    gen = torch.Generator(device=dev).manual_seed(42 + rank)
    eng.grid.uniform_(-1.0, 1.0, generator=gen)
    eng.grid[:, 0], eng.grid[:, -1], eng.grid[:, :, 0], eng.grid[:, :, -1] = 0, 0, 0, 0
    if rank == 0:
        eng.grid[0] = 0
    if rank == world - 1:
        eng.grid[-1] = 0
    eng.run(2)  # warm
    if world > 1:
        dist.barrier(device_ids=[local])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    eng.run(args.sweeps)
    e1.record()
    torch.cuda.synchronize()
    sec = torch.tensor([e0.elapsed_time(e1) / 1e3], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(sec, op=dist.ReduceOp.MAX)
    if rank == 0:
        lups = args.sweeps * n ** 3
        print(json.dumps({"metric": "GS z-pipeline MLUP/s (fp64)", "kernel": args.kernel,
                          "value": lups / float(sec.item()) / 1e6, "n_gpus": world, "n": n,
                          "sweeps": args.sweeps, "scaling": "strong"}), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
