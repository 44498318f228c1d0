"""z-slab decomposition (multi-GPU Jacobi): the exchange logic of
paper_1004_1741_b200.slabs on CPU with gloo (world size 2, oracle compute),
and on one GPU with several slabs (C ABI sb_jacobi_slabs and SlabEngine)."""

import os
import socket

import numpy as np
import pytest

import oracle
from conftest import make_input, sha

from paper_1004_1741_b200.slabs import slab_layout


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def cpu_compute(a, b):
    """Oracle stand-in for sb_jacobi_planes: T sweeps of the local grid,
    keep only the output planes (test infrastructure)."""
    import torch

    def compute(src, dst, nkl, k_lo, k_hi, sweeps):
        if k_hi <= k_lo:
            return
        out = oracle.run_serial("jacobi", src.numpy(), sweeps, a, b)
        dst[k_lo:k_hi] = torch.from_numpy(out[k_lo:k_hi])

    return compute


def _gloo_worker(rank, world, port, spec, iters, depth, a, b, result_path):
    import torch
    import torch.distributed as dist

    from paper_1004_1741_b200.slabs import SlabEngine

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = make_input(spec)
    eng = SlabEngine(g.ni, g.nj, g.nk, depth, rank, world, cpu_compute(a, b),
                     like=torch.empty(0, dtype=torch.float64))
    eng.load_global(g.data)
    eng.run(iters)
    owned = eng.owned().contiguous()
    if rank == 0:
        parts = [owned]
        for r in range(1, world):
            lo, hi, _, _ = slab_layout(g.nk, world, r, depth)
            t = torch.empty((hi - lo, g.nj + 2, g.ni + 2), dtype=torch.float64)
            dist.recv(t, src=r)
            parts.append(t)
        np.save(result_path, torch.cat(parts).numpy())
    else:
        dist.send(owned, dst=0)
    dist.destroy_process_group()


@pytest.mark.parametrize("shape,iters,depth,coeffs", [
    ((12, 10, 16), 7, 2, (0.0, 1 / 6)),
    ((9, 8, 13), 5, 3, (0.5, 0.1)),
    ((6, 6, 4), 4, 1, (0.5, 0.1)),
])
def test_gloo_two_ranks_bitwise_equal_single_grid(tmp_path, shape, iters, depth, coeffs):
    import torch.multiprocessing as mp

    spec = {"shape": list(shape), "pattern": "random", "seed": 5, "lo": -1.0, "hi": 1.0}
    out = tmp_path / "owned.npy"
    mp.start_processes(_gloo_worker, args=(2, _free_port(), spec, iters, depth, *coeffs, str(out)),
                       nprocs=2, join=True, start_method="spawn")
    got = np.load(out)
    want = oracle.run_serial("jacobi", make_input(spec).data, iters, *coeffs)[1:-1]
    assert sha(got) == sha(want)


def test_slab_layout_ghosts():
    assert slab_layout(10, 1, 0, 4) == (1, 11, 1, 1)
    assert slab_layout(10, 3, 1, 2) == (5, 8, 2, 2)
    assert slab_layout(10, 3, 0, 2)[2] == 1 and slab_layout(10, 3, 2, 2)[3] == 1


@pytest.mark.gpu
@pytest.mark.parametrize("nslabs,depth,iters", [(2, 2, 7), (3, 4, 9), (4, 1, 5), (2, 8, 16),
                                                (10, 4, 11), (5, 8, 13)])
def test_c_abi_slabs_on_one_gpu(nslabs, depth, iters):
    """sb_jacobi_slabs, every slab on GPU 0 with its own stream (the fused
    exchange: edge launches store into the neighbours' ghost planes; the last
    two cases have slabs exactly `depth` planes thick, so every owned plane
    goes to both neighbours, and a shallower final period) == the oracle."""
    import ctypes

    import torch

    from paper_1004_1741_b200 import _lib

    lib = _lib.load()
    spec = {"shape": [64, 30, 40], "pattern": "random", "seed": 9, "lo": 0.0, "hi": 1.0}
    g = make_input(spec)
    want = oracle.run_serial("jacobi", g.data, iters, 0.0, 1 / 6)
    bufs, scr = [], []
    for s in range(nslabs):
        lo, hi, gl, gh = slab_layout(g.nk, nslabs, s, depth)
        part = torch.from_numpy(np.ascontiguousarray(g.data[lo - gl:hi + gh])).cuda()
        bufs.append(part)
        scr.append(torch.empty_like(part))
    devs = (ctypes.c_int * nslabs)(*([0] * nslabs))
    pa = (ctypes.c_void_p * nslabs)(*[t.data_ptr() for t in bufs])
    pb = (ctypes.c_void_p * nslabs)(*[t.data_ptr() for t in scr])
    streams = [torch.cuda.Stream() for _ in range(nslabs)]
    ps = (ctypes.c_void_p * nslabs)(*[s.cuda_stream for s in streams])
    res = ctypes.c_int(-1)
    _lib.check(lib.sb_jacobi_slabs(nslabs, devs, pa, pb, g.ni, g.nj, g.nk, iters, 0.0, 1 / 6, depth,
                                   ps, ctypes.byref(res)))
    owned = []
    for s in range(nslabs):
        lo, hi, gl, gh = slab_layout(g.nk, nslabs, s, depth)
        t = (scr if res.value else bufs)[s]
        owned.append(t[gl:gl + hi - lo].cpu().numpy())
    assert sha(np.concatenate(owned)) == sha(want[1:-1])


@pytest.mark.gpu
def test_slab_engine_single_rank_matches_oracle():
    import torch

    from paper_1004_1741_b200.slabs import SlabEngine, gpu_compute

    spec = {"shape": [62, 20, 33], "pattern": "random", "seed": 4, "lo": 0.0, "hi": 1.0}
    g = make_input(spec)
    eng = SlabEngine(g.ni, g.nj, g.nk, 4, 0, 1, gpu_compute(g.ni, g.nj, 0.0, 1 / 6),
                     like=torch.empty(0, dtype=torch.float64, device="cuda"))
    eng.load_global(g.data)
    eng.run(10)
    torch.cuda.synchronize()
    want = oracle.run_serial("jacobi", g.data, 10, 0.0, 1 / 6)
    assert sha(eng.owned().cpu().numpy()) == sha(want[1:-1])


@pytest.mark.gpu
@pytest.mark.parametrize("world,shape,iters,depth", [
    (3, (62, 20, 36), 10, 4),
    (2, (128, 70, 40), 9, 4),
    (4, (254, 33, 50), 7, 3),
    (2, (64, 40, 24), 16, 8),
])
def test_rank_engines_in_lockstep_on_one_gpu(world, shape, iters, depth):
    """The bench's N > 1 compute path on real launches: `world` rank engines
    (edge launches, ghost layout, interior launch through sb_jacobi_planes)
    advance period by period on one GPU; the NCCL exchange is replaced by
    copies of the same plane ranges between the engines."""
    import torch

    from paper_1004_1741_b200.slabs import SlabEngine, gpu_compute

    spec = {"shape": list(shape), "pattern": "random", "seed": 9, "lo": -1.0, "hi": 1.0}
    g = make_input(spec)
    a, b = 0.25, 0.125
    like = torch.empty(0, dtype=torch.float64, device="cuda")
    engs = [SlabEngine(g.ni, g.nj, g.nk, depth, r, world, gpu_compute(g.ni, g.nj, a, b), like=like)
            for r in range(world)]
    for e in engs:
        e.load_global(g.data)
    left = iters
    while left > 0:
        t = min(depth, left)
        for e in engs:
            e.edges(t)
        for r, e in enumerate(engs):  # what SlabEngine._exchange sends and receives
            dst, d, hi = e.bufs[e.cur ^ 1], e.depth, e.glo + e.n_own
            if r + 1 < world:
                up = engs[r + 1]
                dst[hi:hi + d].copy_(up.bufs[up.cur ^ 1][up.glo:up.glo + d])
            if r > 0:
                dn = engs[r - 1]
                dhi = dn.glo + dn.n_own
                dst[0:e.glo].copy_(dn.bufs[dn.cur ^ 1][dhi - d:dhi])
        for e in engs:
            e.interior(t)
        left -= t
    torch.cuda.synchronize()
    want = oracle.run_serial("jacobi", g.data, iters, a, b)
    got = np.concatenate([e.owned().cpu().numpy() for e in engs])
    assert sha(got) == sha(want[1:-1])


# ---------------------------------------------------------------------------
# Gauss-Seidel cross-slab pipeline


def cpu_gs_compute(kernel, b):
    """Oracle stand-in for sb_gs on a local slab grid (test infrastructure)."""
    import torch

    def compute(grid, nkl, sweeps):
        out = oracle.run_serial(kernel, grid.numpy(), sweeps, 0.0, b)
        grid.copy_(torch.from_numpy(out))

    return compute


def _gloo_gs_worker(rank, world, port, spec, iters, kernel, b, result_path):
    import torch
    import torch.distributed as dist

    from paper_1004_1741_b200.slabs import GsSlabEngine, gs_slab_layout

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = make_input(spec)
    eng = GsSlabEngine(g.ni, g.nj, g.nk, rank, world, cpu_gs_compute(kernel, b),
                       like=torch.empty(0, dtype=torch.float64))
    eng.load_global(g.data)
    eng.run(iters)
    owned = eng.owned().contiguous()
    if rank == 0:
        parts = [owned]
        for r in range(1, world):
            lo, hi = gs_slab_layout(g.nk, world, r)
            t = torch.empty((hi - lo, g.nj + 2, g.ni + 2), dtype=torch.float64)
            dist.recv(t, src=r)
            parts.append(t)
        np.save(result_path, torch.cat(parts).numpy())
    else:
        dist.send(owned, dst=0)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,shape,iters,kernel", [
    (2, (12, 10, 9), 6, "gs-naive"),
    (3, (9, 8, 7), 5, "gs-interleaved"),
    (3, (6, 5, 3), 4, "gs-naive"),
])
def test_gloo_gs_pipeline_bitwise_equal_single_grid(tmp_path, world, shape, iters, kernel):
    """The GS z-pipeline (real exchange code, oracle compute) on world ranks
    equals the serial reference sweep bit for bit."""
    import torch.multiprocessing as mp

    spec = {"shape": list(shape), "pattern": "random", "seed": 8, "lo": -1.0, "hi": 1.0}
    out = tmp_path / "owned.npy"
    mp.start_processes(_gloo_gs_worker, args=(world, _free_port(), spec, iters, kernel, 1 / 6,
                                              str(out)),
                       nprocs=world, join=True, start_method="spawn")
    got = np.load(out)
    want = oracle.run_serial(kernel, make_input(spec).data, iters, 0.0, 1 / 6)[1:-1]
    assert sha(got) == sha(want)


def test_gs_slab_layout_matches_c_abi():
    import ctypes

    from paper_1004_1741_b200 import _lib
    from paper_1004_1741_b200.errors import PartitionError
    from paper_1004_1741_b200.slabs import gs_slab_layout

    lib = _lib.load()
    for nk, n in ((10, 3), (7, 7), (64, 5), (2048, 8)):
        for s in range(n):
            lo, hi = ctypes.c_int64(), ctypes.c_int64()
            _lib.check(lib.sb_gs_slab_layout(nk, n, s, ctypes.byref(lo), ctypes.byref(hi)))
            assert (lo.value, hi.value) == gs_slab_layout(nk, n, s)
    lo, hi = ctypes.c_int64(), ctypes.c_int64()
    with pytest.raises(PartitionError):
        _lib.check(lib.sb_gs_slab_layout(3, 4, 0, ctypes.byref(lo), ctypes.byref(hi)))


@pytest.mark.gpu
@pytest.mark.parametrize("nslabs,iters,kernel", [(2, 5, "gs-naive"), (3, 7, "gs-interleaved"),
                                                 (5, 3, "gs-naive")])
def test_c_abi_gs_slabs_on_one_gpu(nslabs, iters, kernel):
    """sb_gs_slabs with every slab on GPU 0 (one stream) == the serial sweep."""
    import ctypes

    import torch

    from paper_1004_1741_b200 import _lib
    from paper_1004_1741_b200.slabs import gs_slab_layout

    lib = _lib.load()
    spec = {"shape": [40, 36, 50], "pattern": "random", "seed": 11, "lo": -1.0, "hi": 1.0}
    g = make_input(spec)
    want = oracle.run_serial(kernel, g.data, iters, 0.0, 1 / 6)
    bufs = []
    for s in range(nslabs):
        lo, hi = gs_slab_layout(g.nk, nslabs, s)
        bufs.append(torch.from_numpy(np.ascontiguousarray(g.data[lo - 1:hi + 1])).cuda())
    st = torch.cuda.Stream()
    devs = (ctypes.c_int * nslabs)(*([0] * nslabs))
    pa = (ctypes.c_void_p * nslabs)(*[t.data_ptr() for t in bufs])
    ps = (ctypes.c_void_p * nslabs)(*([st.cuda_stream] * nslabs))
    _lib.check(lib.sb_gs_slabs(nslabs, devs, pa, g.ni, g.nj, g.nk, iters, 1 / 6,
                               _lib.KERNEL_IDS[kernel], ps))
    owned = [t[1:-1].cpu().numpy() for t in bufs]
    assert sha(np.concatenate(owned)) == sha(want[1:-1])


@pytest.mark.gpu
def test_gs_slab_engine_single_rank_matches_oracle():
    import torch

    from paper_1004_1741_b200.slabs import GsSlabEngine, gpu_gs_compute

    spec = {"shape": [62, 20, 33], "pattern": "random", "seed": 4, "lo": -1.0, "hi": 1.0}
    g = make_input(spec)
    eng = GsSlabEngine(g.ni, g.nj, g.nk, 0, 1, gpu_gs_compute(g.ni, g.nj, 1 / 6, "gs-naive"),
                       like=torch.empty(0, dtype=torch.float64, device="cuda"))
    eng.load_global(g.data)
    eng.run(6)
    torch.cuda.synchronize()
    want = oracle.run_serial("gs-naive", g.data, 6, 0.0, 1 / 6)
    assert sha(eng.owned().cpu().numpy()) == sha(want[1:-1])


@pytest.mark.gpu
@pytest.mark.parametrize("world,shape,iters,kernel", [
    (3, (62, 20, 36), 5, "gs-naive"),
    (2, (128, 70, 40), 4, "gs-interleaved"),
    (4, (30, 33, 50), 6, "gs-naive"),
])
def test_gs_rank_engines_in_pipeline_order_on_one_gpu(world, shape, iters, kernel):
    """The torchrun GS engine's compute path on real launches: `world` rank
    engines sweep their slabs (sb_gs on the local grid with its ghost planes)
    in pipeline order on one GPU; the plane sends are replaced by copies."""
    import torch

    from paper_1004_1741_b200.slabs import GsSlabEngine, gpu_gs_compute

    spec = {"shape": list(shape), "pattern": "random", "seed": 11, "lo": -1.0, "hi": 1.0}
    g = make_input(spec)
    b = 1 / 6
    like = torch.empty(0, dtype=torch.float64, device="cuda")
    engs = [GsSlabEngine(g.ni, g.nj, g.nk, r, world, gpu_gs_compute(g.ni, g.nj, b, kernel), like=like)
            for r in range(world)]
    for e in engs:
        e.load_global(g.data)
    for _ in range(iters):
        for r, e in enumerate(engs):  # rank r's sweep s after rank r-1's sweep s
            if r > 0:
                dn = engs[r - 1]
                e.grid[0].copy_(dn.grid[dn.nkl])          # new values of the plane below
            if r + 1 < world:
                up = engs[r + 1]
                e.grid[e.nkl + 1].copy_(up.grid[1])       # old values of the plane above
            e.compute(e.grid, e.nkl, 1)
    torch.cuda.synchronize()
    want = oracle.run_serial(kernel, g.data, iters, 0.0, b)
    got = np.concatenate([e.owned().cpu().numpy() for e in engs])
    assert sha(got) == sha(want[1:-1])


@pytest.mark.gpu
@pytest.mark.parametrize("nslabs", [2, 8])
def test_c_abi_gs_slabs_full_size(nslabs):
    """Config 5's shape (512^3, U[-1,1)): the GS z-pipeline over `nslabs`
    plane slabs on one GPU == sb_gs on the whole grid, bitwise (4 sweeps)."""
    import ctypes

    import torch

    from paper_1004_1741_b200 import _lib
    from paper_1004_1741_b200.slabs import gs_slab_layout

    lib = _lib.load()
    n, iters = 512, 4
    x = torch.rand((n + 2, n + 2, n + 2), dtype=torch.float64, device="cuda",
                   generator=torch.Generator(device="cuda").manual_seed(5)) * 2 - 1
    x[0], x[-1], x[:, 0], x[:, -1], x[:, :, 0], x[:, :, -1] = 0, 0, 0, 0, 0, 0
    bufs = []
    for s in range(nslabs):
        lo, hi = gs_slab_layout(n, nslabs, s)
        bufs.append(x[lo - 1:hi + 1].clone())
    whole = x.clone()
    _lib.check(lib.sb_gs(whole.data_ptr(), n, n, n, iters, 1 / 6, 1, None))
    _lib.check(lib.sb_sync(None))
    st = torch.cuda.Stream()
    devs = (ctypes.c_int * nslabs)(*([0] * nslabs))
    pa = (ctypes.c_void_p * nslabs)(*[t.data_ptr() for t in bufs])
    ps = (ctypes.c_void_p * nslabs)(*([st.cuda_stream] * nslabs))
    _lib.check(lib.sb_gs_slabs(nslabs, devs, pa, n, n, n, iters, 1 / 6, 1, ps))
    torch.cuda.synchronize()
    for s in range(nslabs):
        lo, hi = gs_slab_layout(n, nslabs, s)
        assert torch.equal(bufs[s][1:-1], whole[lo:hi]), s


def _gs_slabs_run(g, nslabs, iters, kernel, streams=None):
    import ctypes

    import torch

    from paper_1004_1741_b200 import _lib
    from paper_1004_1741_b200.slabs import gs_slab_layout

    lib = _lib.load()
    bufs = []
    for s in range(nslabs):
        lo, hi = gs_slab_layout(g.nk, nslabs, s)
        bufs.append(torch.from_numpy(np.ascontiguousarray(g.data[lo - 1:hi + 1])).cuda())
    st = torch.cuda.Stream()
    devs = (ctypes.c_int * nslabs)(*([0] * nslabs))
    pa = (ctypes.c_void_p * nslabs)(*[t.data_ptr() for t in bufs])
    ps = (ctypes.c_void_p * nslabs)(*(streams or [st.cuda_stream] * nslabs))
    _lib.check(lib.sb_gs_slabs(nslabs, devs, pa, g.ni, g.nj, g.nk, iters, 1 / 6,
                               _lib.KERNEL_IDS[kernel], ps))
    return np.concatenate([t[1:-1].cpu().numpy() for t in bufs])


@pytest.mark.gpu
@pytest.mark.parametrize("shape,nslabs,iters,kernel", [
    ((40, 33, 10), 4, 9, "gs-naive"),          # slabs of 3, 3, 2, 2 planes: one partial tile each
    ((64, 17, 23), 3, 11, "gs-interleaved"),   # 8, 8, 7 planes; > 3 sweep windows
    ((39, 20, 18), 2, 5, "gs-naive"),          # odd ni: the launch-per-sweep fallback
    ((130, 70, 61), 8, 4, "gs-interleaved"),   # 8 slabs in one launch
])
def test_gs_fused_slabs_edge_cases(shape, nslabs, iters, kernel):
    """The fused z-pipeline (one launch for the slabs of a GPU, edge-plane
    chunks pushed into the neighbours' ghost planes) == the serial sweep."""
    spec = {"shape": list(shape), "pattern": "random", "seed": 21, "lo": -1.0, "hi": 1.0}
    g = make_input(spec)
    want = oracle.run_serial(kernel, g.data, iters, 0.0, 1 / 6)
    assert sha(_gs_slabs_run(g, nslabs, iters, kernel)) == sha(want[1:-1])


@pytest.mark.gpu
def test_gs_slabs_sharing_a_device_need_one_stream():
    import torch

    g = make_input({"shape": [16, 8, 8], "pattern": "random", "seed": 1, "lo": 0.0, "hi": 1.0})
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    with pytest.raises(ValueError):
        _gs_slabs_run(g, 2, 1, "gs-naive", streams=[s1.cuda_stream, s2.cuda_stream])


@pytest.mark.gpu
@pytest.mark.parametrize("nslabs", [2, 8])
def test_config5_gs_slabs_vs_reference_hash(hashed_cases, nslabs):
    """BASELINE config 5 (512^3, U[-1,1), 100 sweeps) as the z-pipeline of
    `nslabs` slabs == the reference's own result."""
    from conftest import coeffs_of

    rec = hashed_cases["cfg5_gsn512_mixed_it100"]
    assert coeffs_of(rec)[1] == 1 / 6
    g = make_input(rec["spec"])
    got = _gs_slabs_run(g, nslabs, rec["iters"], rec["kernel"])
    full = g.data.copy()
    full[1:-1] = got
    assert sha(full) == rec["output_sha256"]
