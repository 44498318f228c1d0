"""Multi-GPU Jacobi: z-slabs with per-time-block halo exchange.

The multi-GPU form of the reference's k-slab threading
(sweeps/threaded.py:28-59: ``partition_blocks(nk, P)`` contiguous k-ranges,
one barrier per sweep).  One process per GPU (torchrun); rank r owns the
interior planes ``partition_blocks(nk, world)[r]`` and stores ``depth``
ghost planes toward each neighbour (``slab_layout``; identical to the C
ABI's ``sb_slab_layout``).  A period advances ``T <= depth`` sweeps:

1. compute the owned planes the neighbours need (``depth`` at each inner
   edge) -- ``sb_jacobi_planes`` restricted to those planes;
2. post the halo exchange (NCCL send/recv of contiguous planes over
   NVLink; on the CPU test path gloo) -- it waits only for step 1;
3. compute the remaining owned planes while the exchange is in flight;
4. wait for the exchange before the next period reads the ghosts.

Each owned plane sees exactly the values a single-grid run would (its
dependence cone after T sweeps stays inside owned + ghost planes), so the
result is bitwise identical to one GPU and to the reference.

The compute step is injected: on GPUs it is ``gpu_compute`` (the library);
the CPU test suite runs the same exchange logic with an oracle compute.
"""

import ctypes

from . import _lib
from .sweeps.plan import partition_blocks


def slab_layout(nk, nslabs, slab, depth):
    """(own_lo, own_hi, ghost_lo, ghost_hi) in global padded plane indices;
    mirrors sb_slab_layout (host.cu) -- tests/test_lib.py pins them equal."""
    lo, hi = partition_blocks(nk, nslabs)[slab]
    ghost_lo = 1 if slab == 0 else depth
    ghost_hi = 1 if slab == nslabs - 1 else depth
    if nslabs > 1 and hi - lo < depth:
        from .errors import PartitionError

        raise PartitionError(f"slab {slab} owns {hi - lo} planes, fewer than depth {depth}")
    return lo + 1, hi + 1, ghost_lo, ghost_hi


def gpu_compute(ni, nj, a, b):
    """compute(src, dst, nk_local, k_out_lo, k_out_hi, sweeps) on the current stream."""
    import torch

    lib = _lib.load()

    def compute(src, dst, nkl, k_lo, k_hi, sweeps):
        if k_hi <= k_lo:
            return
        stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        _lib.check(lib.sb_jacobi_planes(src.data_ptr(), dst.data_ptr(), ni, nj, nkl, k_lo, k_hi,
                                        sweeps, a, b, stream))

    return compute


class SlabEngine:
    """This rank's slab of a z-slab decomposed Jacobi run."""

    def __init__(self, ni, nj, nk, depth, rank, world, compute, like, group=None):
        """like: a tensor whose device/dtype the slab buffers use."""
        import torch

        self.ni, self.nj, self.nk, self.depth = ni, nj, nk, depth
        self.rank, self.world, self.group = rank, world, group
        self.compute = compute
        self.own_lo, self.own_hi, self.glo, self.ghi = slab_layout(nk, world, rank, depth)
        self.n_own = self.own_hi - self.own_lo
        self.nkl = self.n_own + self.glo + self.ghi - 2  # local interior planes
        self.k0 = self.own_lo - self.glo                # global index of local plane 0
        shape = (self.nkl + 2, nj + 2, ni + 2)
        self.bufs = [torch.empty(shape, dtype=like.dtype, device=like.device),
                     torch.empty(shape, dtype=like.dtype, device=like.device)]
        self.cur = 0
        self.pending = []

    # -- data movement ---------------------------------------------------------------
    @property
    def field(self):
        """Local buffer holding the current field (owned planes exact)."""
        return self.bufs[self.cur]

    def load_global(self, global_data):
        """Fill both buffers from the global padded grid (host or device)."""
        import torch

        part = global_data[self.k0:self.k0 + self.nkl + 2]
        if not torch.is_tensor(part):
            part = torch.from_numpy(part)
        self.bufs[0].copy_(part)
        self.bufs[1].copy_(self.bufs[0])
        self.cur = 0

    def owned(self):
        """View of the owned planes of the current field."""
        return self.field[self.glo:self.glo + self.n_own]

    # -- one period -----------------------------------------------------------------
    def _exchange(self, dst):
        import torch.distributed as dist

        ops = []
        d = self.depth
        hi = self.glo + self.n_own
        if self.rank + 1 < self.world:
            ops.append(dist.P2POp(dist.isend, dst[hi - d:hi], self.rank + 1, self.group))
            ops.append(dist.P2POp(dist.irecv, dst[hi:hi + d], self.rank + 1, self.group))
        if self.rank > 0:
            ops.append(dist.P2POp(dist.isend, dst[self.glo:self.glo + d], self.rank - 1, self.group))
            ops.append(dist.P2POp(dist.irecv, dst[0:self.glo], self.rank - 1, self.group))
        return dist.batch_isend_irecv(ops) if ops else []

    def wait(self):
        for w in self.pending:
            w.wait()
        self.pending = []

    def ranges(self):
        """(edge_lo, edge_hi, interior) local plane ranges of one period: the
        owned planes a neighbour's ghosts are fed from, and the rest."""
        lo, hi, d = self.glo, self.glo + self.n_own, self.depth
        inner_lo = min(lo + d, hi) if self.rank > 0 else lo
        inner_hi = max(hi - d, inner_lo) if self.rank + 1 < self.world else hi
        return (lo, inner_lo), (inner_hi, hi), (inner_lo, inner_hi)

    def edges(self, sweeps):
        """Phase 1 of a period: the ghost-feeding edge planes, src -> dst."""
        assert 1 <= sweeps <= self.depth
        src, dst = self.bufs[self.cur], self.bufs[self.cur ^ 1]
        (a0, a1), (b0, b1), _ = self.ranges()
        if self.rank > 0:
            self.compute(src, dst, self.nkl, a0, a1, sweeps)
        if self.rank + 1 < self.world:
            self.compute(src, dst, self.nkl, b0, b1, sweeps)

    def interior(self, sweeps):
        """Phase 3 of a period: the remaining owned planes; flips the buffers."""
        src, dst = self.bufs[self.cur], self.bufs[self.cur ^ 1]
        _, _, (c0, c1) = self.ranges()
        self.compute(src, dst, self.nkl, c0, c1, sweeps)
        self.cur ^= 1

    def period(self, sweeps):
        """Advance `sweeps` (<= depth) sweeps; the exchange stays in flight
        until the next period (or wait())."""
        self.wait()
        self.edges(sweeps)
        self.pending = list(self._exchange(self.bufs[self.cur ^ 1])) if self.world > 1 else []
        self.interior(sweeps)

    def run(self, iters):
        left = iters
        while left > 0:
            t = min(self.depth, left)
            self.period(t)
            left -= t
        self.wait()


# ---------------------------------------------------------------------------
# Gauss-Seidel: the cross-GPU z-pipeline (reference pipeline GS,
# sweeps/threaded.py:62-96 / PAPER:336-345, with slabs of planes as stages).


def gs_slab_layout(nk, nslabs, slab):
    """(own_lo, own_hi) global padded planes of a GS slab; its local grid
    holds global planes own_lo-1 .. own_hi (one ghost plane each side).
    Mirrors sb_gs_slab_layout (host.cu)."""
    lo, hi = partition_blocks(nk, nslabs)[slab]
    return lo + 1, hi + 1


def gpu_gs_compute(ni, nj, b, kernel):
    """compute(grid, nk_local, sweeps): in-place GS sweeps of a local grid on
    the current stream (sb_gs; the ghost planes are its k-halo)."""
    import torch

    lib = _lib.load()
    kid = _lib.KERNEL_IDS[kernel]

    def compute(grid, nkl, sweeps):
        stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        _lib.check(lib.sb_gs(grid.data_ptr(), ni, nj, nkl, sweeps, b, kid, stream))

    return compute


class GsSlabEngine:
    """This rank's slab of a pipelined multi-GPU Gauss-Seidel run.

    Sweep s of rank g needs rank g-1's last plane after sweep s (the new
    D values of the lexicographic order) and rank g+1's first plane after
    sweep s-1 (the old U values); with those as the ghost planes, one
    in-place sweep of the local grid equals the global sweep on the owned
    planes, bitwise.  Ranks therefore advance as a pipeline, one plane sent
    each way per sweep and interface (S/(S+G-1) efficient for S sweeps)."""

    def __init__(self, ni, nj, nk, rank, world, compute, like, group=None):
        import torch

        self.ni, self.nj, self.nk = ni, nj, nk
        self.rank, self.world, self.group = rank, world, group
        self.compute = compute
        self.own_lo, self.own_hi = gs_slab_layout(nk, world, rank)
        self.nkl = self.own_hi - self.own_lo
        self.grid = torch.empty((self.nkl + 2, nj + 2, ni + 2), dtype=like.dtype, device=like.device)
        self.sends = []

    def load_global(self, global_data):
        """Fill the local grid (owned + ghost planes) from the global grid."""
        import torch

        part = global_data[self.own_lo - 1:self.own_hi + 1]
        if not torch.is_tensor(part):
            part = torch.from_numpy(part)
        self.grid.copy_(part)

    def owned(self):
        return self.grid[1:self.nkl + 1]

    def sweep(self, s, last=False):
        """Sweep number s (0-based) of this slab; `last`: no sweep follows, so
        the first plane is not sent down (nothing would receive it)."""
        import torch.distributed as dist

        recvs = []
        if self.rank > 0:  # new values of the plane below
            recvs.append(dist.irecv(self.grid[0], self.rank - 1, self.group))
        if self.rank + 1 < self.world and s > 0:  # old values of the plane above
            recvs.append(dist.irecv(self.grid[self.nkl + 1], self.rank + 1, self.group))
        for w in self.sends + recvs:  # sent planes are overwritten by this sweep
            w.wait()
        self.compute(self.grid, self.nkl, 1)
        self.sends = []
        if self.rank + 1 < self.world:
            self.sends.append(dist.isend(self.grid[self.nkl], self.rank + 1, self.group))
        if self.rank > 0 and not last:
            self.sends.append(dist.isend(self.grid[1], self.rank - 1, self.group))

    def run(self, iters):
        if self.world == 1:
            if iters:
                self.compute(self.grid, self.nkl, iters)
            return
        for s in range(iters):
            self.sweep(s, last=(s == iters - 1))
        for w in self.sends:
            w.wait()
        self.sends = []
