// host.cu -- host-buffer entry point and the z-slab decomposition driver.
//
// sb_run_host is the whole reference `sweeps.run(plan, g)` contract in one
// synchronous call on host memory (the numpy path of the Python drop-in).
//
// The z-slab functions are the multi-GPU form of the reference's k-slab
// threading (sweeps/threaded.py:28-59, partition_blocks at :39): slab s owns
// the contiguous interior planes partition_blocks(nk, nslabs)[s] and keeps
// `depth` ghost planes per inner side, so `depth` fused sweeps can run
// between two halo exchanges (the overlapped-halo form of the paper's
// per-time-block exchange).  Each period computes the ghost-feeding edge
// planes first, then the slab interior while the edges travel to the
// neighbours (cudaMemcpyPeerAsync over NVLink, or a device copy when two
// slabs share a GPU).  Results are bitwise identical to the single-grid run.
#include <cuda_runtime.h>

#include <algorithm>
#include <functional>
#include <cstring>
#include <mutex>
#include <utility>
#include <vector>

#include "../../include/stencil_b200.h"
#include "sb_internal.h"
#include "jacobi_tb.cuh"

namespace sb {
int gs_check_error(cudaStream_t st);

// cached device buffers + stream per device for sb_run_host
struct HostCtx {
    double* g = nullptr;
    double* s = nullptr;
    size_t cap = 0;  // doubles per buffer
    cudaStream_t st = nullptr;
};
static std::mutex g_host_mu;
static HostCtx g_host[64];

// true when kernels on device a can store into device b's memory (the same
// device, or peer access possible both ways)
bool peer_reachable(int a, int b) {
    if (a == b) return true;
    int ab = 0, ba = 0;
    cudaDeviceCanAccessPeer(&ab, a, b);
    cudaDeviceCanAccessPeer(&ba, b, a);
    return ab && ba;
}

// Streams and events created for the duration of one driver call, destroyed
// on every return path (error returns included).
struct CallHandles {
    std::vector<std::pair<int, cudaStream_t>> streams;
    std::vector<std::pair<int, cudaEvent_t>> events;
    cudaError_t stream(int dev, cudaStream_t* out) {
        cudaError_t e = cudaSetDevice(dev);
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(out, cudaStreamNonBlocking);
        if (e == cudaSuccess) streams.emplace_back(dev, *out);
        return e;
    }
    cudaError_t event(int dev, cudaEvent_t* out) {
        cudaError_t e = cudaSetDevice(dev);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(out, cudaEventDisableTiming);
        if (e == cudaSuccess) events.emplace_back(dev, *out);
        return e;
    }
    ~CallHandles() {
        for (auto& x : events) {
            cudaSetDevice(x.first);
            cudaEventDestroy(x.second);
        }
        for (auto& x : streams) {
            cudaSetDevice(x.first);
            cudaStreamDestroy(x.second);
        }
    }
    CallHandles() = default;
    CallHandles(const CallHandles&) = delete;
    CallHandles& operator=(const CallHandles&) = delete;
};

// partition_blocks semantics (reference sweeps/plan.py:106-120)
static void part(int64_t extent, int count, int idx, int64_t* lo, int64_t* hi) {
    const int64_t base = extent / count, rem = extent % count;
    *lo = idx * base + std::min<int64_t>(idx, rem);
    *hi = *lo + base + (idx < rem ? 1 : 0);
}

}  // namespace sb

using namespace sb;

extern "C" {

int sb_run_host(int kernel, double* host_grid, int64_t ni, int64_t nj, int64_t nk, int64_t iters,
                double a, double b, int depth, int device) {
    clear_error();
    DeviceGuard guard;
    int rc = check_dims(ni, nj, nk);
    if (rc) return rc;
    if (iters < 0) return fail(SB_ERR_PLAN, "iter_end must be >= 0, got %lld", (long long)iters);
    if (kernel < SB_KERNEL_JACOBI || kernel > SB_KERNEL_GS_INTERLEAVED)
        return fail(SB_ERR_PLAN, "unknown kernel %d", kernel);
    if (kernel == SB_KERNEL_JACOBI && (depth < 1 || depth > sb_max_depth()))
        return fail(SB_ERR_PLAN, "depth must be in [1, %d], got %d", sb_max_depth(), depth);
    if (!host_grid) return fail(SB_ERR_ARGUMENT, "null pointer");
    if (iters == 0) return SB_OK;
    int ndev = sb_device_count();
    if (ndev < 1) return fail(SB_ERR_NODEVICE, "no CUDA device");
    if (device < 0 || device >= ndev || device >= 64)
        return fail(SB_ERR_ARGUMENT, "device %d out of range (%d visible)", device, ndev);
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");

    std::lock_guard<std::mutex> lk(g_host_mu);
    HostCtx& H = g_host[device];
    const size_t count = size_t(ni + 2) * size_t(nj + 2) * size_t(nk + 2);
    const size_t bytes = count * sizeof(double);
    if (!H.st && (e = cudaStreamCreateWithFlags(&H.st, cudaStreamNonBlocking)) != cudaSuccess)
        return cuda_fail(e, "cudaStreamCreate");
    const bool two = (kernel == SB_KERNEL_JACOBI);
    if (H.cap < count || (two && !H.s)) {
        if (H.g) cudaFree(H.g);
        if (H.s) cudaFree(H.s);
        H.g = H.s = nullptr;
        H.cap = 0;
        if ((e = cudaMalloc(&H.g, bytes)) != cudaSuccess) return cuda_fail(e, "cudaMalloc(grid)");
        if (two && (e = cudaMalloc(&H.s, bytes)) != cudaSuccess) {
            cudaFree(H.g);
            H.g = nullptr;
            return cuda_fail(e, "cudaMalloc(scratch)");
        }
        H.cap = count;
    }
    if ((e = cudaMemcpyAsync(H.g, host_grid, bytes, cudaMemcpyHostToDevice, H.st)) != cudaSuccess)
        return cuda_fail(e, "H2D copy");
    const double* result = H.g;
    if (kernel == SB_KERNEL_JACOBI) {
        int in_s = 0;
        rc = sb_jacobi(H.g, H.s, ni, nj, nk, iters, a, b, depth, H.st, &in_s);
        if (rc) return rc;
        result = in_s ? H.s : H.g;
    } else {
        rc = sb_gs(H.g, ni, nj, nk, iters, b, kernel, H.st);
        if (rc) return rc;
    }
    if ((e = cudaMemcpyAsync(host_grid, result, bytes, cudaMemcpyDeviceToHost, H.st)) != cudaSuccess)
        return cuda_fail(e, "D2H copy");
    if ((e = cudaStreamSynchronize(H.st)) != cudaSuccess) return cuda_fail(e, "sweep execution");
    if (kernel != SB_KERNEL_JACOBI) return gs_check_error(H.st);
    return SB_OK;
}

// Pipelined host-buffer batch: entry i's upload overlaps entry i-1's sweeps
// and entry i-2's download (two device slots, one stream each for H2D,
// sweeps and D2H; PCIe is full duplex and the copy engines are separate), so
// a stream of grids moves at max(H2D, sweeps, D2H) per grid instead of the
// sum.  Ordering: D2H(i) completes before H2D(i+2) starts (same slot), so an
// entry may repeat the pointer of an entry >= 2 places earlier and then starts
// from that entry's result; adjacent repeats are rejected.
// Device slots of the batch pipeline.  Three slots let entry i+1's upload
// run during entry i's sweeps while entry i-1 downloads (PCIe Gen5 is full
// duplex: 55.6 GB/s up, 53.9 down, 94.6 together on B200), so a batch moves
// at about max(H2D, sweeps, D2H, duplex) per grid; two slots (if memory is
// short) serialise each upload behind the download two entries back.
constexpr int kBatchSlots = 3;
struct BatchCtx {
    double* g[kBatchSlots] = {};
    double* s[kBatchSlots] = {};
    int nslots = 0;
    size_t cap = 0;
    bool two = false;
    cudaStream_t st[3] = {nullptr, nullptr, nullptr};  // H2D, sweeps, D2H
    cudaEvent_t up[kBatchSlots], done[kBatchSlots], down[kBatchSlots];
    bool ev = false;
};
static BatchCtx g_batch[64];

static void batch_free(BatchCtx& B) {
    B.nslots = 0;
    for (int i = 0; i < kBatchSlots; ++i) {
        if (B.g[i]) cudaFree(B.g[i]);
        if (B.s[i]) cudaFree(B.s[i]);
        B.g[i] = B.s[i] = nullptr;
    }
    B.cap = 0;
}

int sb_release_caches(int device) {
    clear_error();
    const int ndev = sb_device_count();
    if (ndev <= 0) return SB_OK;
    DeviceGuard guard;
    for (int d = 0; d < std::min(ndev, 64); ++d) {
        if (device >= 0 && d != device) continue;
        bool holds;
        {
            std::lock_guard<std::mutex> lk(g_host_mu);
            holds = g_batch[d].nslots > 0 || g_host[d].g || g_host[d].s;
        }
        // devices without cached buffers are not touched (no new contexts)
        if (!holds && !gs_holds(d) && !jacobi_holds(d)) continue;
        cudaError_t e = cudaSetDevice(d);
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        if (e != cudaSuccess) return cuda_fail(e, "sb_release_caches");
        std::lock_guard<std::mutex> lk(g_host_mu);
        batch_free(g_batch[d]);
        HostCtx& H = g_host[d];
        if (H.g) cudaFree(H.g);
        if (H.s) cudaFree(H.s);
        H.g = H.s = nullptr;
        H.cap = 0;
        gs_release(d);
        jacobi_release(d);
    }
    return SB_OK;
}

int sb_run_host_batch(int kernel, double* const* host_grids, int count, int64_t ni, int64_t nj,
                      int64_t nk, int64_t iters, double a, double b, int depth, int device) {
    clear_error();
    DeviceGuard guard;
    int rc = check_dims(ni, nj, nk);
    if (rc) return rc;
    if (iters < 0) return fail(SB_ERR_PLAN, "iter_end must be >= 0, got %lld", (long long)iters);
    if (kernel < SB_KERNEL_JACOBI || kernel > SB_KERNEL_GS_INTERLEAVED)
        return fail(SB_ERR_PLAN, "unknown kernel %d", kernel);
    if (kernel == SB_KERNEL_JACOBI && (depth < 1 || depth > sb_max_depth()))
        return fail(SB_ERR_PLAN, "depth must be in [1, %d], got %d", sb_max_depth(), depth);
    if (count < 0 || (count > 0 && !host_grids)) return fail(SB_ERR_ARGUMENT, "bad grid list");
    for (int i = 0; i < count; ++i) {
        if (!host_grids[i]) return fail(SB_ERR_ARGUMENT, "null grid pointer at %d", i);
        if (i > 0 && host_grids[i] == host_grids[i - 1])
            return fail(SB_ERR_ARGUMENT, "entries %d and %d are the same grid", i - 1, i);
    }
    if (iters == 0 || count == 0) return SB_OK;
    int ndev = sb_device_count();
    if (ndev < 1) return fail(SB_ERR_NODEVICE, "no CUDA device");
    if (device < 0 || device >= ndev || device >= 64)
        return fail(SB_ERR_ARGUMENT, "device %d out of range (%d visible)", device, ndev);
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");

    std::lock_guard<std::mutex> lk(g_host_mu);
    BatchCtx& B = g_batch[device];
    const size_t cells = size_t(ni + 2) * size_t(nj + 2) * size_t(nk + 2);
    const size_t bytes = cells * sizeof(double);
    const bool two = (kernel == SB_KERNEL_JACOBI);
    if (!B.st[0]) {
        for (int i = 0; i < 3; ++i)
            if ((e = cudaStreamCreateWithFlags(&B.st[i], cudaStreamNonBlocking)) != cudaSuccess)
                return cuda_fail(e, "cudaStreamCreate");
    }
    if (!B.ev) {
        for (int i = 0; i < kBatchSlots; ++i) {
            if ((e = cudaEventCreateWithFlags(&B.up[i], cudaEventDisableTiming)) != cudaSuccess ||
                (e = cudaEventCreateWithFlags(&B.done[i], cudaEventDisableTiming)) != cudaSuccess ||
                (e = cudaEventCreateWithFlags(&B.down[i], cudaEventDisableTiming)) != cudaSuccess)
                return cuda_fail(e, "cudaEventCreate");
        }
        B.ev = true;
    }
    if (B.cap < cells || (two && !B.two)) {
        batch_free(B);
        for (int i = 0; i < kBatchSlots; ++i) {
            if ((e = cudaMalloc(&B.g[i], bytes)) != cudaSuccess ||
                (two && (e = cudaMalloc(&B.s[i], bytes)) != cudaSuccess)) {
                cudaGetLastError();
                if (i >= 2) break;  // two slots still pipeline
                batch_free(B);
                return cuda_fail(e, "cudaMalloc(batch slots)");
            }
            B.nslots = i + 1;
        }
        if (B.nslots < kBatchSlots) {  // drop a half-allocated slot
            const int i = B.nslots;
            if (B.g[i]) cudaFree(B.g[i]);
            if (B.s[i]) cudaFree(B.s[i]);
            B.g[i] = B.s[i] = nullptr;
        }
        B.cap = cells;
        B.two = two;
    }
    const int ns = B.nslots;
    cudaStream_t h2d = B.st[0], comp = B.st[1], d2h = B.st[2];
    for (int i = 0; i < count; ++i) {
        const int sl = i % ns;
        // the slot's previous entry has been downloaded
        if (i >= ns && (e = cudaStreamWaitEvent(h2d, B.down[sl], 0)) != cudaSuccess)
            return cuda_fail(e, "cudaStreamWaitEvent");
        // an entry repeating the grid of an entry still in flight starts from
        // that entry's result (entries up to i-ns are already ordered above)
        for (int j = std::max(0, i - ns + 1); j < i; ++j)
            if (host_grids[j] == host_grids[i] &&
                (e = cudaStreamWaitEvent(h2d, B.down[j % ns], 0)) != cudaSuccess)
                return cuda_fail(e, "cudaStreamWaitEvent");
        if ((e = cudaMemcpyAsync(B.g[sl], host_grids[i], bytes, cudaMemcpyHostToDevice, h2d)) !=
                cudaSuccess ||
            (e = cudaEventRecord(B.up[sl], h2d)) != cudaSuccess ||
            (e = cudaStreamWaitEvent(comp, B.up[sl], 0)) != cudaSuccess)
            return cuda_fail(e, "H2D copy");
        const double* result = B.g[sl];
        if (two) {
            int in_s = 0;
            rc = sb_jacobi(B.g[sl], B.s[sl], ni, nj, nk, iters, a, b, depth, comp, &in_s);
            if (rc) return rc;
            result = in_s ? B.s[sl] : B.g[sl];
        } else {
            rc = sb_gs(B.g[sl], ni, nj, nk, iters, b, kernel, comp);
            if (rc) return rc;
        }
        if ((e = cudaEventRecord(B.done[sl], comp)) != cudaSuccess ||
            (e = cudaStreamWaitEvent(d2h, B.done[sl], 0)) != cudaSuccess ||
            (e = cudaMemcpyAsync(host_grids[i], result, bytes, cudaMemcpyDeviceToHost, d2h)) !=
                cudaSuccess ||
            (e = cudaEventRecord(B.down[sl], d2h)) != cudaSuccess)
            return cuda_fail(e, "D2H copy");
    }
    if ((e = cudaStreamSynchronize(d2h)) != cudaSuccess) return cuda_fail(e, "batch execution");
    if ((e = cudaStreamSynchronize(comp)) != cudaSuccess) return cuda_fail(e, "batch execution");
    if (!two) return gs_check_error(comp);
    return SB_OK;
}

int sb_jacobi_planes(const double* src, double* dst, int64_t ni, int64_t nj, int64_t nk,
                     int64_t k_out_lo, int64_t k_out_hi, int sweeps, double a, double b,
                     void* stream) {
    clear_error();
    int rc = check_dims(ni, nj, nk);
    if (rc) return rc;
    if (sweeps < 1 || sweeps > sb_max_depth())
        return fail(SB_ERR_PLAN, "sweeps per block must be in [1, %d], got %d", sb_max_depth(), sweeps);
    if (k_out_lo < 1 || k_out_hi > nk + 1 || k_out_lo > k_out_hi)
        return fail(SB_ERR_ARGUMENT, "output planes [%lld, %lld) outside [1, %lld]", (long long)k_out_lo,
                    (long long)k_out_hi, (long long)nk);
    if (!src || !dst || src == dst) return fail(SB_ERR_ARGUMENT, "need two distinct buffers");
    return jacobi_block(src, dst, (int)ni, (int)nj, (int)nk, (int)k_out_lo, (int)k_out_hi, sweeps, a, b,
                        static_cast<cudaStream_t>(stream));
}

int sb_slab_layout(int64_t nk, int nslabs, int slab, int depth, int64_t* own_lo, int64_t* own_hi,
                   int64_t* ghost_lo, int64_t* ghost_hi) {
    clear_error();
    if (nslabs < 1 || nslabs > nk)
        return fail(SB_ERR_PARTITION, "cannot split nk=%lld planes into %d slabs", (long long)nk, nslabs);
    if (slab < 0 || slab >= nslabs) return fail(SB_ERR_ARGUMENT, "slab %d of %d", slab, nslabs);
    if (depth < 1 || depth > sb_max_depth()) return fail(SB_ERR_PLAN, "depth %d", depth);
    int64_t lo, hi;
    part(nk, nslabs, slab, &lo, &hi);
    *own_lo = lo + 1;  // padded global plane indices
    *own_hi = hi + 1;
    *ghost_lo = (slab == 0) ? 1 : depth;
    *ghost_hi = (slab == nslabs - 1) ? 1 : depth;
    if (nslabs > 1 && hi - lo < depth)
        return fail(SB_ERR_PARTITION, "slab %d owns %lld planes, fewer than depth %d", slab,
                    (long long)(hi - lo), depth);
    return SB_OK;
}

int sb_jacobi_slabs(int nslabs, const int* devices, double* const* slabs, double* const* scratch,
                    int64_t ni, int64_t nj, int64_t nk, int64_t iters, double a, double b, int depth,
                    void* const* streams, int* result_in_scratch) {
    clear_error();
    DeviceGuard guard;
    int rc = check_dims(ni, nj, nk);
    if (rc) return rc;
    if (iters < 0) return fail(SB_ERR_PLAN, "iter_end must be >= 0, got %lld", (long long)iters);
    if (!devices || !slabs || !scratch || !streams || !result_in_scratch)
        return fail(SB_ERR_ARGUMENT, "null pointer");
    struct Slab {
        int dev;
        double* buf[2];
        cudaStream_t st, comm;
        int64_t own_lo, own_hi, glo, ghi, nkl;  // nkl: local interior planes
        cudaEvent_t edge, start, sent_up, sent_dn;
    };
    std::vector<Slab> S(nslabs);
    for (int s = 0; s < nslabs; ++s) {
        if ((rc = sb_slab_layout(nk, nslabs, s, depth, &S[s].own_lo, &S[s].own_hi, &S[s].glo, &S[s].ghi)))
            return rc;
        S[s].dev = devices[s];
        S[s].buf[0] = slabs[s];
        S[s].buf[1] = scratch[s];
        S[s].st = static_cast<cudaStream_t>(streams[s]);
        S[s].nkl = (S[s].own_hi - S[s].own_lo) + S[s].glo + S[s].ghi - 2;
        if (!slabs[s] || !scratch[s] || slabs[s] == scratch[s])
            return fail(SB_ERR_ARGUMENT, "slab %d needs two distinct buffers", s);
    }
    *result_in_scratch = 0;
    if (iters == 0) return SB_OK;
    const int64_t nip = ni + 2, plane = nip * (nj + 2);
    const size_t pbytes = size_t(plane) * sizeof(double);
    cudaError_t e;
    CallHandles handles;  // this call's streams and events (DeviceGuard restores the device after it)
    // peer access where the slabs live on different GPUs
    for (int s = 0; s < nslabs; ++s) {
        if ((e = cudaSetDevice(S[s].dev)) != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
        for (int t = 0; t < nslabs; ++t)
            if (S[t].dev != S[s].dev) {
                int can = 0;
                cudaDeviceCanAccessPeer(&can, S[s].dev, S[t].dev);
                if (can) {
                    e = cudaDeviceEnablePeerAccess(S[t].dev, 0);
                    if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                    else if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceEnablePeerAccess");
                }
            }
        // both buffers must carry the Dirichlet halo (and the initial ghosts)
        if ((rc = halo_copy(S[s].buf[0], S[s].buf[1], (int)ni, (int)nj, (int)S[s].nkl, S[s].st))) return rc;
    }
    int cur = 0;  // buffer index holding the current field
    // Fused exchange (every slab TMA-addressable): per slab and period, the
    // `depth` edge planes on each inner side are computed first by launches
    // whose threads also write them into the neighbours' ghost planes (peer
    // memory over NVLink between GPUs; JacPeers) -- no separate copies -- then
    // the interior by the plain kernel.  Period p of slab s waits for period
    // p-1 of s-1 and s+1: its ghosts were written there, and they read the
    // planes this period's edge launches overwrite.  Events alternate by
    // period parity so that a wait never lands on the same period.
    // (the kernels store into the neighbours' buffers: slabs on different
    // GPUs need peer access between them, else the copy-based exchange runs)
    bool fused = (ni % 2 == 0);
    for (int s = 0; s < nslabs; ++s) {
        fused = fused && tma_ok(S[s].buf[0], ni) && tma_ok(S[s].buf[1], ni);
        if (s + 1 < nslabs) fused = fused && peer_reachable(S[s].dev, S[s + 1].dev);
    }
    if (fused) {
        std::vector<cudaEvent_t> pev[2];
        for (int par = 0; par < 2; ++par) {
            pev[par].assign(nslabs, nullptr);
            for (int s = 0; s < nslabs; ++s)
                if ((e = handles.event(S[s].dev, &pev[par][s])) != cudaSuccess)
                    return cuda_fail(e, "cudaEventCreate");
        }
        rc = SB_OK;
        int64_t period = 0;
        for (int64_t done = 0; done < iters && rc == SB_OK; ++period) {
            const int T = (int)std::min<int64_t>(depth, iters - done);
            const int par = int(period & 1);
            for (int s = 0; s < nslabs && rc == SB_OK; ++s) {
                Slab& X = S[s];
                cudaSetDevice(X.dev);
                if (period > 0) {
                    if (s > 0) cudaStreamWaitEvent(X.st, pev[par ^ 1][s - 1], 0);
                    if (s + 1 < nslabs) cudaStreamWaitEvent(X.st, pev[par ^ 1][s + 1], 0);
                }
                const int64_t lo = X.glo, hi = X.glo + (X.own_hi - X.own_lo);  // owned, local padded
                JacPeers pe;
                memset(&pe, 0, sizeof pe);
                if (s + 1 < nslabs) {  // top `depth` owned planes -> the slab above's planes [0, depth)
                    pe.buf[0] = S[s + 1].buf[cur ^ 1];
                    pe.k0[0] = int(hi - depth);
                    pe.k1[0] = int(hi);
                    pe.off[0] = int(depth - hi);
                }
                if (s > 0) {  // bottom `depth` owned planes -> the slab below's [Y.hi, Y.hi + depth)
                    const Slab& Y = S[s - 1];
                    pe.buf[1] = Y.buf[cur ^ 1];
                    pe.k0[1] = int(lo);
                    pe.k1[1] = int(lo + depth);
                    pe.off[1] = int(Y.glo + (Y.own_hi - Y.own_lo) - lo);
                }
                const JacPeers* pp = (pe.buf[0] || pe.buf[1]) ? &pe : nullptr;
                const int64_t elo = (s > 0) ? std::min<int64_t>(lo + depth, hi) : lo;
                const int64_t ehi = (s + 1 < nslabs) ? std::max<int64_t>(hi - depth, elo) : hi;
                const double* src = X.buf[cur];
                double* dst = X.buf[cur ^ 1];
                const int nkl = (int)X.nkl;
                if (elo > lo)
                    rc = jacobi_block(src, dst, (int)ni, (int)nj, nkl, (int)lo, (int)elo, T, a, b, X.st, pp);
                if (rc == SB_OK && hi > ehi)
                    rc = jacobi_block(src, dst, (int)ni, (int)nj, nkl, (int)ehi, (int)hi, T, a, b, X.st, pp);
                if (rc == SB_OK && ehi > elo)
                    rc = jacobi_block(src, dst, (int)ni, (int)nj, nkl, (int)elo, (int)ehi, T, a, b, X.st);
                if (rc == SB_OK) cudaEventRecord(pev[par][s], X.st);
            }
            cur ^= 1;
            done += T;
        }
        for (int s = 0; s < nslabs; ++s) {
            cudaSetDevice(S[s].dev);
            if ((e = cudaStreamSynchronize(S[s].st)) != cudaSuccess && rc == SB_OK)
                rc = cuda_fail(e, "slab sweeps");
        }
        *result_in_scratch = cur;
        return rc;
    }
    // copy-based exchange: a comm stream and four events per slab
    for (int s = 0; s < nslabs; ++s) {
        if ((e = handles.stream(S[s].dev, &S[s].comm)) != cudaSuccess) return cuda_fail(e, "cudaStreamCreate");
        for (cudaEvent_t* ev : {&S[s].edge, &S[s].start, &S[s].sent_up, &S[s].sent_dn})
            if ((e = handles.event(S[s].dev, ev)) != cudaSuccess) return cuda_fail(e, "cudaEventCreate");
    }
    bool first = true;
    for (int64_t done = 0; done < iters;) {
        const int T = (int)std::min<int64_t>(depth, iters - done);
        // 1. per slab: edge planes, then interior
        for (int s = 0; s < nslabs; ++s) {
            Slab& X = S[s];
            cudaSetDevice(X.dev);
            if (!first) {  // last period's incoming/outgoing copies must be done
                if (s > 0) cudaStreamWaitEvent(X.st, S[s - 1].sent_up, 0);
                if (s + 1 < nslabs) cudaStreamWaitEvent(X.st, S[s + 1].sent_dn, 0);
                cudaStreamWaitEvent(X.st, X.sent_up, 0);
                cudaStreamWaitEvent(X.st, X.sent_dn, 0);
            }
            cudaEventRecord(X.start, X.st);
            const double* src = X.buf[cur];
            double* dst = X.buf[cur ^ 1];
            const int64_t lo = X.glo, hi = X.glo + (X.own_hi - X.own_lo);  // owned, local padded
            const int64_t elo = (s > 0) ? std::min<int64_t>(lo + depth, hi) : lo;
            const int64_t ehi = (s + 1 < nslabs) ? std::max<int64_t>(hi - depth, elo) : hi;
            if (s > 0 && (rc = jacobi_block(src, dst, (int)ni, (int)nj, (int)X.nkl, (int)lo, (int)elo, T, a, b, X.st)))
                return rc;
            if (s + 1 < nslabs &&
                (rc = jacobi_block(src, dst, (int)ni, (int)nj, (int)X.nkl, (int)ehi, (int)hi, T, a, b, X.st)))
                return rc;
            cudaEventRecord(X.edge, X.st);
            if ((rc = jacobi_block(src, dst, (int)ni, (int)nj, (int)X.nkl, (int)elo, (int)ehi, T, a, b, X.st)))
                return rc;
        }
        // 2. exchange: top `depth` owned planes up, bottom `depth` owned planes down
        for (int s = 0; s < nslabs; ++s) {
            Slab& X = S[s];
            cudaSetDevice(X.dev);
            double* xd = X.buf[cur ^ 1];
            const int64_t hi = X.glo + (X.own_hi - X.own_lo);
            if (s + 1 < nslabs) {
                Slab& Y = S[s + 1];
                cudaStreamWaitEvent(X.comm, X.edge, 0);
                cudaStreamWaitEvent(X.comm, Y.start, 0);
                // X planes [hi-depth, hi) -> Y local planes [0, depth)
                e = cudaMemcpyPeerAsync(Y.buf[cur ^ 1], Y.dev, xd + (hi - depth) * plane, X.dev,
                                        depth * pbytes, X.comm);
                if (e != cudaSuccess) return cuda_fail(e, "halo exchange (up)");
                cudaEventRecord(X.sent_up, X.comm);
            }
            if (s > 0) {
                Slab& Y = S[s - 1];
                cudaStreamWaitEvent(X.comm, X.edge, 0);
                cudaStreamWaitEvent(X.comm, Y.start, 0);
                // X planes [glo, glo+depth) -> Y local planes [Y.hi, Y.hi+depth)
                const int64_t yhi = Y.glo + (Y.own_hi - Y.own_lo);
                e = cudaMemcpyPeerAsync(Y.buf[cur ^ 1] + yhi * plane, Y.dev, xd + X.glo * plane, X.dev,
                                        depth * pbytes, X.comm);
                if (e != cudaSuccess) return cuda_fail(e, "halo exchange (down)");
                cudaEventRecord(X.sent_dn, X.comm);
            }
        }
        cur ^= 1;
        first = false;
        done += T;
    }
    for (int s = 0; s < nslabs; ++s) {
        cudaSetDevice(S[s].dev);
        if ((e = cudaStreamSynchronize(S[s].comm)) != cudaSuccess) return cuda_fail(e, "exchange");
        if ((e = cudaStreamSynchronize(S[s].st)) != cudaSuccess) return cuda_fail(e, "slab sweeps");
    }
    *result_in_scratch = cur;
    return SB_OK;
}

// Gauss-Seidel across slabs: the cross-GPU z-pipeline form of the reference's
// pipeline GS (sweeps/threaded.py:62-96).  Slab g owns the
// interior planes partition_blocks(nk, nslabs)[g]; its local grid holds them
// between two ghost planes that act as its k-halo: below, slab g-1's last
// plane after the current sweep (new values: the D neighbour of the
// lexicographic order); above, slab g+1's first plane after the previous
// sweep (old values: U).  One in-place GS sweep of the local grid is then
// exactly the global sweep on the owned planes, so results are bitwise
// identical to one grid.  Sweep s of slab g waits for sweep s of slab g-1
// and sweep s-1 of slab g+1: the slabs advance as a pipeline, S/(S+G-1)
// efficient for S sweeps on G slabs.
int sb_gs_slab_layout(int64_t nk, int nslabs, int slab, int64_t* own_lo, int64_t* own_hi) {
    clear_error();
    if (nslabs < 1 || nslabs > nk)
        return fail(SB_ERR_PARTITION, "cannot split nk=%lld planes into %d slabs", (long long)nk, nslabs);
    if (slab < 0 || slab >= nslabs) return fail(SB_ERR_ARGUMENT, "slab %d of %d", slab, nslabs);
    if (!own_lo || !own_hi) return fail(SB_ERR_ARGUMENT, "null pointer");
    int64_t lo, hi;
    part(nk, nslabs, slab, &lo, &hi);
    *own_lo = lo + 1;  // padded global plane indices
    *own_hi = hi + 1;
    return SB_OK;
}

int sb_gs_slabs(int nslabs, const int* devices, double* const* slabs, int64_t ni, int64_t nj,
                int64_t nk, int64_t iters, double b, int kernel, void* const* streams) {
    clear_error();
    DeviceGuard guard;
    int rc = check_dims(ni, nj, nk);
    if (rc) return rc;
    if (iters < 0) return fail(SB_ERR_PLAN, "iter_end must be >= 0, got %lld", (long long)iters);
    if (kernel != SB_KERNEL_GS_NAIVE && kernel != SB_KERNEL_GS_INTERLEAVED)
        return fail(SB_ERR_PLAN, "sb_gs_slabs runs the Gauss-Seidel kernels, got %d", kernel);
    if (!devices || !slabs || !streams) return fail(SB_ERR_ARGUMENT, "null pointer");
    struct Slab {
        int dev;
        double* g;
        cudaStream_t st;
        int64_t nkl;                   // owned planes (local interior)
        cudaEvent_t done, got_lo, got_hi;  // sweep finished / ghost copies finished
    };
    std::vector<Slab> S(nslabs);
    for (int g = 0; g < nslabs; ++g) {
        int64_t lo, hi;
        if ((rc = sb_gs_slab_layout(nk, nslabs, g, &lo, &hi))) return rc;
        if (!slabs[g]) return fail(SB_ERR_ARGUMENT, "null slab %d", g);
        S[g].dev = devices[g];
        S[g].g = slabs[g];
        S[g].st = static_cast<cudaStream_t>(streams[g]);
        S[g].nkl = hi - lo;
    }
    if (iters == 0) return SB_OK;
    const int64_t plane = (ni + 2) * (nj + 2);
    const size_t pbytes = size_t(plane) * sizeof(double);
    cudaError_t e;
    // slabs sharing a device share its stream (one launch per device)
    for (int g = 0; g < nslabs; ++g)
        for (int h = 0; h < g; ++h)
            if (S[h].dev == S[g].dev && S[h].st != S[g].st)
                return fail(SB_ERR_ARGUMENT, "slabs %d and %d share device %d but not a stream", h, g,
                            S[g].dev);
    for (int g = 0; g < nslabs; ++g) {
        if ((e = cudaSetDevice(S[g].dev)) != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
        for (int h : {g - 1, g + 1})
            if (h >= 0 && h < nslabs && S[h].dev != S[g].dev) {
                int can = 0;
                cudaDeviceCanAccessPeer(&can, S[g].dev, S[h].dev);
                if (can) {
                    e = cudaDeviceEnablePeerAccess(S[h].dev, 0);
                    if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                    else if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceEnablePeerAccess");
                }
            }
    }
    // the fused pipeline: one persistent launch per device, edge-plane chunks
    // pushed into the neighbours' ghost planes as they are stored
    {
        std::vector<int64_t> nks(nslabs);
        std::vector<double*> grids(nslabs);
        for (int g = 0; g < nslabs; ++g) {
            nks[g] = S[g].nkl;
            grids[g] = S[g].g;
        }
        rc = gs_slabs_fused(nslabs, devices, grids.data(), nks.data(), (int)ni, (int)nj, iters, b, kernel,
                            streams);
        if (rc != SB_ERR_PLAN) return rc;
        clear_error();
    }
    // not eligible (odd ni, unaligned slabs, > 8 slabs on a device): one
    // sb_gs launch per slab and sweep, ghost planes copied between them
    CallHandles handles;
    for (int g = 0; g < nslabs; ++g)
        for (cudaEvent_t* ev : {&S[g].done, &S[g].got_lo, &S[g].got_hi})
            if ((e = handles.event(S[g].dev, ev)) != cudaSuccess) return cuda_fail(e, "cudaEventCreate");
    for (int64_t sw = 0; sw < iters; ++sw) {
        for (int g = 0; g < nslabs; ++g) {
            Slab& X = S[g];
            cudaSetDevice(X.dev);
            if (g > 0) {  // ghost below: slab g-1's last plane after this sweep
                Slab& Y = S[g - 1];
                cudaStreamWaitEvent(X.st, Y.done, 0);
                if ((e = cudaMemcpyPeerAsync(X.g, X.dev, Y.g + Y.nkl * plane, Y.dev, pbytes, X.st)) !=
                    cudaSuccess)
                    return cuda_fail(e, "ghost copy (below)");
                cudaEventRecord(X.got_lo, X.st);
                // slab g-1 read this slab's first plane (old) before it changes
                if (sw > 0) cudaStreamWaitEvent(X.st, Y.got_hi, 0);
            }
            if (g + 1 < nslabs && sw > 0) {  // ghost above: slab g+1's first plane, previous sweep
                Slab& Y = S[g + 1];
                cudaStreamWaitEvent(X.st, Y.done, 0);
                if ((e = cudaMemcpyPeerAsync(X.g + (X.nkl + 1) * plane, X.dev, Y.g + plane, Y.dev, pbytes,
                                             X.st)) != cudaSuccess)
                    return cuda_fail(e, "ghost copy (above)");
                cudaEventRecord(X.got_hi, X.st);
                // slab g+1 copied this slab's last plane (previous sweep) before it changes
                cudaStreamWaitEvent(X.st, Y.got_lo, 0);
            }
            if ((rc = sb_gs(X.g, ni, nj, X.nkl, 1, b, kernel, X.st))) return rc;
            cudaEventRecord(X.done, X.st);
        }
    }
    rc = SB_OK;
    for (int g = 0; g < nslabs; ++g) {
        cudaSetDevice(S[g].dev);
        if ((e = cudaStreamSynchronize(S[g].st)) != cudaSuccess && rc == SB_OK)
            rc = cuda_fail(e, "slab sweeps");
    }
    return rc;
}

// The whole `run(plan, g)` contract over several GPUs: the grid (host or
// device memory, UVA) is cut into z-slabs per partition_blocks, one per
// entry of `devices`, scattered (with ghost planes), swept by the slab
// drivers above and gathered back.  The multi-GPU form of the reference's
// run_threaded_jacobi (k-slabs, threaded.py:28-59) and run_pipeline_gs
// (pipelined stages, threaded.py:62-96).
int sb_run_multi(int kernel, double* grid, int64_t ni, int64_t nj, int64_t nk, int64_t iters,
                 double a, double b, int depth, int ndev, const int* devices) {
    clear_error();
    DeviceGuard guard;
    int rc = check_dims(ni, nj, nk);
    if (rc) return rc;
    if (iters < 0) return fail(SB_ERR_PLAN, "iter_end must be >= 0, got %lld", (long long)iters);
    if (kernel < SB_KERNEL_JACOBI || kernel > SB_KERNEL_GS_INTERLEAVED)
        return fail(SB_ERR_PLAN, "unknown kernel %d", kernel);
    const bool jac = (kernel == SB_KERNEL_JACOBI);
    if (jac && (depth < 1 || depth > sb_max_depth()))
        return fail(SB_ERR_PLAN, "depth must be in [1, %d], got %d", sb_max_depth(), depth);
    if (!grid || !devices) return fail(SB_ERR_ARGUMENT, "null pointer");
    if (ndev < 1) return fail(SB_ERR_ARGUMENT, "need at least one device, got %d", ndev);
    if (ndev > nk)
        return fail(SB_ERR_PARTITION, "cannot split nk=%lld planes into %d slabs", (long long)nk, ndev);
    const int visible = sb_device_count();
    if (visible < 1) return fail(SB_ERR_NODEVICE, "no CUDA device");
    for (int s = 0; s < ndev; ++s)
        if (devices[s] < 0 || devices[s] >= visible)
            return fail(SB_ERR_ARGUMENT, "device %d out of range (%d visible)", devices[s], visible);
    if (iters == 0) return SB_OK;
    // ghost width: the requested depth, capped by the thinnest inner slab
    // (results are identical for every depth)
    int T = 1;
    if (jac) {
        T = depth;
        if (ndev > 1) T = (int)std::min<int64_t>(T, nk / ndev);
        if (ni % 2) T = 1;  // the slab blocks have no pitched path (odd rows: one sweep each)
        T = std::max(T, 1);
    }
    const int64_t plane = (ni + 2) * (nj + 2);
    const size_t pbytes = size_t(plane) * sizeof(double);
    struct Part {
        int64_t lo, hi, glo, ghi, nkl;  // owned global padded planes; ghosts; local interior planes
        double* buf[2] = {nullptr, nullptr};
    };
    std::vector<Part> P(ndev);
    std::vector<int> devs(devices, devices + ndev);
    std::vector<cudaStream_t> st(ndev, nullptr);
    std::vector<cudaStream_t> dev_stream(visible, nullptr);  // one stream per device (GS needs it)
    cudaError_t e = cudaSuccess;
    auto cleanup = [&]() {
        for (int s = 0; s < ndev; ++s) {
            cudaSetDevice(devs[s]);
            for (double* p : P[s].buf)
                if (p) cudaFree(p);
        }
        for (int d = 0; d < visible; ++d)
            if (dev_stream[d]) {
                cudaSetDevice(d);
                cudaStreamDestroy(dev_stream[d]);
            }
    };
    struct Cleanup {
        std::function<void()> f;
        ~Cleanup() { f(); }
    } on_exit{cleanup};
    for (int s = 0; s < ndev; ++s) {
        Part& X = P[s];
        if (jac) {
            if ((rc = sb_slab_layout(nk, ndev, s, T, &X.lo, &X.hi, &X.glo, &X.ghi))) return rc;
        } else {
            if ((rc = sb_gs_slab_layout(nk, ndev, s, &X.lo, &X.hi))) return rc;
            X.glo = X.ghi = 1;
        }
        X.nkl = (X.hi - X.lo) + X.glo + X.ghi - 2;
        if ((e = cudaSetDevice(devs[s])) != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
        if (!dev_stream[devs[s]] &&
            (e = cudaStreamCreateWithFlags(&dev_stream[devs[s]], cudaStreamNonBlocking)) != cudaSuccess)
            return cuda_fail(e, "cudaStreamCreate");
        st[s] = dev_stream[devs[s]];
        const size_t bytes = size_t(X.nkl + 2) * pbytes;
        for (int i = 0; i < (jac ? 2 : 1); ++i)
            if ((e = cudaMalloc(&X.buf[i], bytes)) != cudaSuccess)
                return cuda_fail(e, "cudaMalloc(slab)");
        // scatter: global planes [lo-glo, hi+ghi) (UVA: host or any device)
        if ((e = cudaMemcpyAsync(X.buf[0], grid + (X.lo - X.glo) * plane, bytes, cudaMemcpyDefault,
                                 st[s])) != cudaSuccess)
            return cuda_fail(e, "scatter copy");
    }
    std::vector<double*> b0(ndev), b1(ndev);
    std::vector<void*> sv(ndev);
    for (int s = 0; s < ndev; ++s) {
        b0[s] = P[s].buf[0];
        b1[s] = P[s].buf[1];
        sv[s] = st[s];
    }
    int in_s = 0;
    if (jac)
        rc = sb_jacobi_slabs(ndev, devs.data(), b0.data(), b1.data(), ni, nj, nk, iters, a, b, T,
                             sv.data(), &in_s);
    else
        rc = sb_gs_slabs(ndev, devs.data(), b0.data(), ni, nj, nk, iters, b, kernel, sv.data());
    if (rc) return rc;
    // gather the owned planes back into the caller's grid
    for (int s = 0; s < ndev; ++s) {
        const Part& X = P[s];
        cudaSetDevice(devs[s]);
        if ((e = cudaMemcpyAsync(grid + X.lo * plane, X.buf[in_s] + X.glo * plane,
                                 size_t(X.hi - X.lo) * pbytes, cudaMemcpyDefault, st[s])) != cudaSuccess)
            return cuda_fail(e, "gather copy");
    }
    for (int s = 0; s < ndev; ++s) {
        cudaSetDevice(devs[s]);
        if ((e = cudaStreamSynchronize(st[s])) != cudaSuccess) return cuda_fail(e, "gather");
    }
    if (!jac) {
        for (int s = 0; s < ndev; ++s) {
            cudaSetDevice(devs[s]);
            if ((rc = gs_check_error(st[s]))) return rc;
        }
    }
    return SB_OK;
}

}  // extern "C"
