// gs.cu -- lexicographic Gauss-Seidel sweeps for sm_100a, bit-exact.
//
// Reference: kernels.py:154-163 (naive), :165-187 (interleaved); the
// engines that preserve the serial order in parallel are the pipeline
// (sweeps/threaded.py:62-96) and the multi-wavefront scheme
// (sweeps/wavefront.py:315-376).
//
// Dependency structure.  Cell (k,j,i) of sweep s reads the sweep-s values
// of its W, S, D neighbours and the sweep-(s-1) values of E, N, U.  Any
// schedule that respects these edges reproduces the serial result bit for
// bit as long as each cell's own arithmetic is identical, so the GPU is
// free to run everything that is not ordered by them concurrently:
//
// * Inside a CTA, a tile of BJ x BK lines (rows j x planes k) is processed
//   by one thread per line.  Line (jl, kl) is skewed by jl+kl steps: at
//   local step t it updates cell i = 1 + t - (jl+kl).  Then S and D were
//   produced one step earlier by the neighbouring lines, N and U are still
//   untouched, and one __syncthreads per step orders everything.  This is
//   the hyperplane wavefront of the paper's pipeline-parallel GS, at cell
//   granularity.
// * The tile's lines plus their halo lines live in shared memory as a ring
//   of column chunks (CW columns x (BJ+2) x (BK+2) lines), filled by one TMA
//   box load per chunk and written back by BK TMA box stores per chunk.
// * Across CTAs, tile (J,K) of sweep s may load chunk c once
//     - tiles (J-1,K), (J,K-1) of sweep s   have stored chunk c (new W/S/D),
//     - tiles (J+1,K), (J,K+1), (J,K) of sweep s-1 have stored chunk c
//       (old N/U/E, not yet overwritten: their sweep-s stores depend on us).
//   Progress counters per (sweep mod R, tile) are published with
//   st.release after the TMA store completed and polled with ld.acquire.
// * Tasks (s, tile) are handed out by an atomic ticket in sweep-major,
//   anti-diagonal (J+K) order, so a task only ever waits on tasks with a
//   smaller ticket, which are already running: deadlock-free on a
//   persistent grid, and successive sweeps pipeline behind each other like
//   the paper's shifted wavefronts.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <algorithm>
#include <vector>

#include "../../include/stencil_b200.h"
#include "sb_internal.h"
#include "sb_ptx.cuh"

namespace sb {

int make_grid_map(CUtensorMap* m, const double* base, int64_t nip, int64_t njp, int64_t nkp, int bw,
                  int bh);
int make_grid_map3(CUtensorMap* m, const double* base, int64_t nip, int64_t njp, int64_t nkp, int bw,
                   int bh, int bd);

struct GsParams {
    int ni, nj, nk;
    int tiles_j, tiles_k, ntiles;
    int nch;               // column chunks per line (ceil((ni+2)/CW))
    int sweeps;            // sweeps in this launch
    long long tasks;       // sweeps * ntiles
    double b;
    int* ticket;           // atomic task counter
    int* prog;             // [R][ntiles] progress (encoded)
    int* err;              // error word (timeout)
    const short2* order;   // ticket -> (J, K) within a sweep
};

template <int BJ_, int BK_, int CW_, int NS_, int MINB_>
struct GsCfg {
    static constexpr int BJ = BJ_, BK = BK_, CW = CW_, NS = NS_, MINB = MINB_;
    static constexpr int NT = BJ * BK;
    static constexpr int LJ = BJ + 2, LK = BK + 2;       // lines incl. halo
    static constexpr int LINES = LJ * LK;
    static constexpr int SLOT = CW * LINES;              // doubles per chunk slot
    static constexpr int SMAX = (BJ - 1) + (BK - 1);     // max line skew
    static constexpr int R = 4;                          // sweep slots for progress
    static constexpr uint32_t BOX_BYTES = uint32_t(SLOT) * 8;
    static constexpr size_t SMEM_BYTES = size_t(NS) * SLOT * 8 + 8 * NS + 64;
    // prefetch distance (steps) before a chunk is first needed
    static constexpr int DPF = CW;
    static_assert((NS - 1) * CW > DPF + SMAX + 2, "too few chunk slots for the skew");
};

// progress encoding: (sweep+1) * (nch+1) + chunks_stored   (0 = nothing)
__device__ __forceinline__ int prog_val(int s, int chunks, int nch) { return (s + 1) * (nch + 1) + chunks; }

template <class C>
__device__ __forceinline__ bool wait_prog(const GsParams& p, int s, int tile, int need_chunks,
                                          volatile int* abort_flag) {
    if (s < 0) return true;
    const int* addr = p.prog + (s % C::R) * p.ntiles + tile;
    const int want = prog_val(s, need_chunks, p.nch);
    if (ld_acquire(addr) >= want) return true;
    const long long t0 = clock64();
    while (ld_acquire(addr) < want) {
        if (*reinterpret_cast<volatile int*>(p.err)) return false;
        if (clock64() - t0 > (1LL << 35)) {  // ~17 s: a dependency never arrived
            atomicExch(p.err, 1);
            return false;
        }
        __nanosleep(64);
    }
    return true;
}

template <class C, bool INTERLEAVED>
__global__ void __launch_bounds__(C::NT, C::MINB)
gs_tile_kernel(const __grid_constant__ CUtensorMap ld_map,
               const __grid_constant__ CUtensorMap st_map, const GsParams p) {
    constexpr int BJ = C::BJ, BK = C::BK, CW = C::CW, NS = C::NS, LJ = C::LJ;
    extern __shared__ __align__(128) double smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + size_t(NS) * C::SLOT);
    __shared__ int s_task[2];
    __shared__ int s_abort;

    const int tid = threadIdx.x;
    const int jl = tid % BJ, kl = tid / BJ;
    const int skew = jl + kl;
    // line index in a chunk slot (halo lines at jl = -1, BJ and kl = -1, BK)
    const int line = (kl + 1) * LJ + (jl + 1);
    const double b = p.b;

    if (tid == 0) {
        for (int s = 0; s < NS; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
        tma_prefetch_desc(&ld_map);
        tma_prefetch_desc(&st_map);
        s_abort = 0;
    }
    uint32_t loads = 0;   // chunk loads issued by this CTA (slot = loads % NS) -- tid 0
    uint32_t waits = 0;   // chunk loads consumed (mirror of loads on all threads)
    int stores_committed = 0;  // tid 0

    while (true) {
        if (tid == 0) {
            int tk = atomicAdd(p.ticket, 1);
            s_task[0] = tk;
        }
        __syncthreads();
        const long long ticket = s_task[0];
        if (ticket >= p.tasks || s_abort) break;
        const int s = (int)(ticket / p.ntiles);
        const short2 jk = p.order[ticket % p.ntiles];
        const int J = jk.x, K = jk.y;
        const int tile = K * p.tiles_j + J;
        const int J0 = 1 + J * BJ, K0 = 1 + K * BK;  // padded origin of the tile's lines
        const int nsteps = p.ni + C::SMAX;            // local steps until every line is done
        const uint32_t base = waits;                  // first chunk load of this task

        // tid 0: dependency-checked chunk loads
        int next_load = 0;  // next chunk to load (tid 0)
        auto issue_loads_upto = [&](int t) -> bool {
            // load every chunk whose due step (c*CW - 2 - DPF) is <= t
            while (next_load < p.nch && next_load * CW - 2 - C::DPF <= t) {
                const int c = next_load;
                bool ok = true;
                ok = ok && (s == 0 || wait_prog<C>(p, s - 1, tile, c + 1, &s_abort));
                if (J > 0) ok = ok && wait_prog<C>(p, s, tile - 1, c + 1, &s_abort);
                if (K > 0) ok = ok && wait_prog<C>(p, s, tile - p.tiles_j, c + 1, &s_abort);
                if (s > 0 && J + 1 < p.tiles_j) ok = ok && wait_prog<C>(p, s - 1, tile + 1, c + 1, &s_abort);
                if (s > 0 && K + 1 < p.tiles_k)
                    ok = ok && wait_prog<C>(p, s - 1, tile + p.tiles_j, c + 1, &s_abort);
                if (!ok) return false;
                fence_proxy_async_global();
                // the slot's previous chunk must have left smem (its store read done)
                bulk_wait_read<0>();
                const uint32_t slot = loads % NS;
                mbar_arrive_expect_tx(&full[slot], C::BOX_BYTES);
                tma_load_3d(smem + size_t(slot) * C::SLOT, &ld_map, c * CW, J0 - 1, K0 - 1, &full[slot]);
                ++loads;
                ++next_load;
            }
            return true;
        };

        if (tid == 0) {
            // a tile may run at most R-1 sweeps ahead of its own oldest unfinished sweep
            bool ok = wait_prog<C>(p, s - (C::R - 1), tile, p.nch, &s_abort);
            ok = ok && issue_loads_upto(-1);
            if (!ok) s_abort = 1;
        }
        __syncthreads();
        if (s_abort) break;

        double w = 0.0;            // own previous (new) value: the W neighbour
        int have = -1;             // highest chunk this thread has waited for (task-local)
        int stored = 0;            // chunks stored (tid 0)
        int published = 0;         // chunks published (tid 0)

        for (int t = 0; t < nsteps; ++t) {
            const int i = 1 + t - skew;  // padded column of this line's cell
            // wait for the chunk holding column i+1 (the leading need of this line)
            {
                const int cneed = min(p.nch - 1, max(0, (i + 1) / CW));
                while (have < cneed) {
                    ++have;
                    const uint32_t ld = base + have;
                    mbar_wait(&full[ld % NS], (ld / NS) & 1);
                }
            }
            const bool active = (i >= 1) && (i <= p.ni) && (J0 + jl <= p.nj) && (K0 + kl <= p.nk);
            if (active) {
                auto at = [&](int ln, int col) -> double* {
                    const int c = col / CW;
                    const uint32_t ld = base + c;
                    return smem + size_t(ld % NS) * C::SLOT + ln * CW + (col - c * CW);
                };
                if (i == 1) w = *at(line, 0);
                const double e = *at(line, i + 1);
                const double sv = *at(line - 1, i);
                const double nv = *at(line + 1, i);
                const double dv = *at(line - LJ, i);
                const double uv = *at(line + LJ, i);
                double x;
                if (INTERLEAVED && p.ni >= 2) {
                    double tmp = __dadd_rn(e, sv);
                    tmp = __dadd_rn(tmp, nv);
                    tmp = __dadd_rn(tmp, dv);
                    tmp = __dadd_rn(tmp, uv);
                    x = __dmul_rn(b, __dadd_rn(w, tmp));
                } else {
                    double acc = __dadd_rn(w, e);
                    acc = __dadd_rn(acc, sv);
                    acc = __dadd_rn(acc, nv);
                    acc = __dadd_rn(acc, dv);
                    acc = __dadd_rn(acc, uv);
                    x = __dmul_rn(b, acc);
                }
                *at(line, i) = x;
                w = x;
            }
            // chunks completed by this step: the trailing line passed their last column
            const int trail_col = 1 + t - C::SMAX;
            const bool last = (t == nsteps - 1);
            int complete = last ? p.nch : max(0, (trail_col + 1) / CW);
            const bool storing = complete > stored;  // uniform across the CTA
            if (storing) fence_proxy_async_smem();
            __syncthreads();
            if (s_abort) break;  // set by tid 0 before this barrier
            if (tid == 0) {
                bool ok = true;
                while (stored < complete) {
                    const uint32_t ld = base + stored;
                    const double* slot = smem + size_t(ld % NS) * C::SLOT;
                    for (int q = 0; q < BK; ++q)
                        tma_store_3d(&st_map, slot + ((q + 1) * LJ + 1) * CW, stored * CW, J0, K0 + q);
                    bulk_commit();
                    ++stores_committed;
                    ++stored;
                }
                // publish what has fully landed (all but the most recent group)
                if (published < stored - 1) {
                    bulk_wait<1>();
                    fence_proxy_async_global();
                    published = stored - 1;
                    st_release(p.prog + (s % C::R) * p.ntiles + tile, prog_val(s, published, p.nch));
                }
                if (last) {
                    bulk_wait<0>();
                    fence_proxy_async_global();
                    published = stored;
                    st_release(p.prog + (s % C::R) * p.ntiles + tile, prog_val(s, published, p.nch));
                }
                ok = issue_loads_upto(t);
                if (!ok) s_abort = 1;
            }
        }
        waits = base + p.nch;
        __syncthreads();
        if (s_abort) break;
    }
    (void)stores_committed;
    if (tid == 0) bulk_wait<0>();
}

// ---------------------------------------------------------------------------
// Odd row pitch (ni+2 odd): TMA cannot describe the grid.  Exact serial
// order by a single thread -- correctness fallback for small odd grids only.
template <bool INTERLEAVED>
__global__ void gs_serial_kernel(double* g, int ni, int nj, int nk, int sweeps, double b) {
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    const int64_t nip = ni + 2, plane = nip * (nj + 2);
    for (int s = 0; s < sweeps; ++s)
        for (int k = 1; k <= nk; ++k)
            for (int j = 1; j <= nj; ++j) {
                double* c = g + k * plane + j * nip;
                if (INTERLEAVED && ni >= 2) {
                    for (int i = 1; i <= ni; ++i) {
                        double tmp = __dadd_rn(c[i + 1], c[i - nip]);
                        tmp = __dadd_rn(tmp, c[i + nip]);
                        tmp = __dadd_rn(tmp, c[i - plane]);
                        tmp = __dadd_rn(tmp, c[i + plane]);
                        c[i] = __dmul_rn(b, __dadd_rn(c[i - 1], tmp));
                    }
                } else {
                    for (int i = 1; i <= ni; ++i) {
                        double acc = __dadd_rn(c[i - 1], c[i + 1]);
                        acc = __dadd_rn(acc, c[i - nip]);
                        acc = __dadd_rn(acc, c[i + nip]);
                        acc = __dadd_rn(acc, c[i - plane]);
                        acc = __dadd_rn(acc, c[i + plane]);
                        c[i] = __dmul_rn(b, acc);
                    }
                }
            }
}

// ---------------------------------------------------------------------------
using GsC = GsCfg<8, 8, 16, 4, 4>;

struct GsScratch {
    int dev = -1;
    int* words = nullptr;      // ticket, err
    int* prog = nullptr;
    size_t prog_cap = 0;
    short2* order = nullptr;
    size_t order_cap = 0;
    int tj = -1, tk = -1;
};
static GsScratch g_gs[16];

int gs_run(double* grid, int ni, int nj, int nk, int64_t iters, double b, int kernel,
           cudaStream_t st) {
    const bool inter = (kernel == SB_KERNEL_GS_INTERLEAVED);
    if (!tma_ok(grid, ni)) {
        for (int64_t done = 0; done < iters;) {
            int n = (int)std::min<int64_t>(iters - done, 1 << 20);
            if (inter) gs_serial_kernel<true><<<1, 32, 0, st>>>(grid, ni, nj, nk, n, b);
            else gs_serial_kernel<false><<<1, 32, 0, st>>>(grid, ni, nj, nk, n, b);
            done += n;
        }
        cudaError_t e = cudaGetLastError();
        return e == cudaSuccess ? SB_OK : cuda_fail(e, "gs_serial launch");
    }
    using C = GsC;
    int dev;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    if (dev >= 16) return fail(SB_ERR_CUDA, "device index %d unsupported", dev);
    GsScratch& S = g_gs[dev];
    int* counters;
    int sms;
    int rc = get_counters(&counters, &sms);
    if (rc) return rc;

    const int tiles_j = (nj + C::BJ - 1) / C::BJ, tiles_k = (nk + C::BK - 1) / C::BK;
    const int ntiles = tiles_j * tiles_k;
    if (!S.words) {
        if ((e = cudaMalloc(&S.words, 64 * sizeof(int))) != cudaSuccess) return cuda_fail(e, "cudaMalloc");
    }
    size_t need = size_t(C::R) * ntiles;
    if (S.prog_cap < need) {
        if (S.prog) cudaFree(S.prog);
        if ((e = cudaMalloc(&S.prog, need * sizeof(int))) != cudaSuccess) return cuda_fail(e, "cudaMalloc");
        S.prog_cap = need;
    }
    if (S.tj != tiles_j || S.tk != tiles_k) {
        // anti-diagonal order: d = J + K ascending, then J ascending
        std::vector<short2> ord;
        ord.reserve(ntiles);
        for (int d = 0; d <= tiles_j + tiles_k - 2; ++d)
            for (int J = 0; J < tiles_j; ++J) {
                int K = d - J;
                if (K >= 0 && K < tiles_k) ord.push_back(make_short2((short)J, (short)K));
            }
        if (S.order_cap < (size_t)ntiles) {
            if (S.order) cudaFree(S.order);
            if ((e = cudaMalloc(&S.order, ntiles * sizeof(short2))) != cudaSuccess)
                return cuda_fail(e, "cudaMalloc");
            S.order_cap = ntiles;
        }
        if ((e = cudaMemcpy(S.order, ord.data(), ntiles * sizeof(short2), cudaMemcpyHostToDevice)) !=
            cudaSuccess)
            return cuda_fail(e, "cudaMemcpy(order)");
        S.tj = tiles_j;
        S.tk = tiles_k;
    }
    if (tiles_j > 32767 || tiles_k > 32767) return fail(SB_ERR_DIMENSION, "grid too large for GS tiling");

    CUtensorMap lmap, smap;
    const int64_t nip = ni + 2, njp = nj + 2, nkp = nk + 2;
    if ((rc = make_grid_map3(&lmap, grid, nip, njp, nkp, C::CW, C::LJ, C::LK))) return rc;
    if ((rc = make_grid_map3(&smap, grid, nip, njp, nkp, C::CW, C::BJ, 1))) return rc;

    static int occ = -1;
    auto kern_n = gs_tile_kernel<C, false>;
    auto kern_i = gs_tile_kernel<C, true>;
    if (occ < 0) {
        for (auto k : {kern_n, kern_i}) {
            e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM_BYTES);
            if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(gs)");
        }
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern_n, C::NT, C::SMEM_BYTES);
        if (e != cudaSuccess || occ < 1) return fail(SB_ERR_CUDA, "gs kernel does not fit");
    }
    GsParams p;
    p.ni = ni;
    p.nj = nj;
    p.nk = nk;
    p.tiles_j = tiles_j;
    p.tiles_k = tiles_k;
    p.ntiles = ntiles;
    p.nch = (ni + 2 + C::CW - 1) / C::CW;
    p.b = b;
    p.ticket = S.words;
    p.err = S.words + 1;
    p.prog = S.prog;
    p.order = S.order;
    // sweeps per launch bounded by the int32 progress encoding
    const int64_t max_sweeps = ((int64_t(1) << 30) / (p.nch + 1)) - 2;
    for (int64_t done = 0; done < iters;) {
        const int n = (int)std::min<int64_t>(iters - done, max_sweeps);
        p.sweeps = n;
        p.tasks = (long long)n * ntiles;
        if ((e = cudaMemsetAsync(S.words, 0, 64 * sizeof(int), st)) != cudaSuccess)
            return cuda_fail(e, "memset");
        if ((e = cudaMemsetAsync(S.prog, 0, need * sizeof(int), st)) != cudaSuccess)
            return cuda_fail(e, "memset");
        const int grid_ctas = (int)std::min<long long>((long long)sms * occ, p.tasks);
        if (inter) kern_i<<<grid_ctas, C::NT, C::SMEM_BYTES, st>>>(lmap, smap, p);
        else kern_n<<<grid_ctas, C::NT, C::SMEM_BYTES, st>>>(lmap, smap, p);
        if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "gs launch");
        done += n;
    }
    return SB_OK;
}

// error word readback (host) -- called by the synchronous entry points
int gs_check_error(cudaStream_t st) {
    int dev;
    if (cudaGetDevice(&dev) != cudaSuccess || dev >= 16 || !g_gs[dev].words) return SB_OK;
    int err = 0;
    cudaError_t e = cudaMemcpyAsync(&err, g_gs[dev].words + 1, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "gs error readback");
    if (err) return fail(SB_ERR_TIMEOUT, "gs: inter-CTA dependency wait timed out");
    return SB_OK;
}

}  // namespace sb

extern "C" int sb_gs(double* grid, int64_t ni, int64_t nj, int64_t nk, int64_t iters, double b,
                     int kernel, void* stream) {
    using namespace sb;
    clear_error();
    int rc = check_dims(ni, nj, nk);
    if (rc) return rc;
    if (iters < 0) return fail(SB_ERR_PLAN, "iter_end must be >= 0, got %lld", (long long)iters);
    if (kernel != SB_KERNEL_GS_NAIVE && kernel != SB_KERNEL_GS_INTERLEAVED)
        return fail(SB_ERR_PLAN, "sb_gs needs a Gauss-Seidel kernel, got %d", kernel);
    if (!grid) return fail(SB_ERR_ARGUMENT, "null pointer");
    if (reinterpret_cast<uintptr_t>(grid) & 7) return fail(SB_ERR_ARGUMENT, "grid must be 8-byte aligned");
    if (iters == 0) return SB_OK;
    return gs_run(grid, (int)ni, (int)nj, (int)nk, iters, b, kernel, static_cast<cudaStream_t>(stream));
}

extern "C" int sb_sync(void* stream) {
    using namespace sb;
    clear_error();
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "stream synchronize");
    return gs_check_error(st);
}
