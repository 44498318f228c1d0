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
// bit as long as each cell's own arithmetic is identical:
//
// * Inside a CTA, a tile of BJ x BK lines (rows j x planes k) is processed
//   by one compute thread per line.  Line (jl, kl) is skewed by jl+kl steps:
//   at local step t it updates cell i = 1 + t - (jl+kl).  S and D were then
//   produced one step earlier by the neighbouring lines, N and U are still
//   untouched, and one named barrier per step (compute warps only) orders
//   everything -- the hyperplane wavefront of the paper's pipeline-parallel
//   GS at cell granularity.
// * The tile's lines plus their halo lines live in shared memory as a ring of
//   column chunks (CW columns x (BJ+2) x (BK+2) lines), filled by TMA box
//   loads and written back by TMA box stores.
// * Warp specialisation: a loader warp polls neighbour progress (with a
//   cache of the last value seen) and issues chunk loads ahead of the
//   compute; a storer warp writes finished chunks back, frees their ring
//   slot once the store has read shared memory and publishes progress once
//   it has landed.  The compute warps only wait on shared-memory mbarriers,
//   at CTA-uniform steps.
// * Across CTAs, tile (J,K) of sweep s may load chunk c once
//     - tiles (J-1,K), (J,K-1) of sweep s          have stored chunk c,
//     - tiles (J+1,K), (J,K+1), (J,K) of sweep s-1 have stored chunk c
//       (old N/U/E, not yet overwritten: their sweep-s stores depend on us).
//   Progress counters per (sweep mod R, tile) are published with st.release
//   after the TMA store completed and polled with ld.acquire.
// * Tasks (sweep, tile) are handed out by an atomic ticket in sweep-major,
//   anti-diagonal (J+K) order, so a task only waits on tasks with smaller
//   tickets, which are already running: deadlock-free on a persistent grid,
//   and successive sweeps pipeline behind each other like the paper's
//   shifted wavefronts.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <cstdlib>
#include <mutex>
#include <type_traits>
#include <utility>
#include <cstdint>
#include <vector>

#include "../../include/stencil_b200.h"
#include "sb_internal.h"
#include "sb_ptx.cuh"

namespace sb {

int make_grid_map3p(CUtensorMap* m, const double* base, int64_t nip, int64_t njp, int64_t nkp,
                    int bw, int bh, int bd, int64_t pitch);

// Slabs.  A launch sweeps one grid, or several z-slabs of one global grid
// (the cross-GPU z-pipeline, sb_gs_slabs): each slab is a local padded grid
// whose planes 0 and nk+1 are ghost planes holding the neighbours' edge
// planes.  Tile (J, 0) of a slab waits for the slab below to have pushed its
// top plane's chunk (sweep s values: D) into the ghost plane below; tile
// (J, last) for the slab above to have pushed its bottom plane's chunk
// (sweep s-1 values: U) into the ghost plane above.  Pushes are plain
// stores by the storer thread (to peer memory when the neighbour is on
// another GPU), published by a system-scope release of a per-(sweep, J)
// flag in the receiving slab's memory -- the same dependency protocol as
// between tiles of one grid, so successive sweeps overlap across slabs (and
// GPUs) as they do across tiles.  The write-after-read hazards on a ghost
// plane are ordered by the chain that already exists: a neighbour's sweep
// s+1 push of chunk c follows its sweep s+1 load of chunk c, which waited
// for this slab's sweep s store (hence load) of chunk c.
constexpr int kGsMaxSlabs = 8;
struct GsSlab {
    int nk;              // interior planes of the slab's local grid
    int tiles_k;         // K tiles of the slab
    int tile0;           // index of tile (0, 0) in the launch's progress arrays
    int* ghost_lo;       // [R][tiles_j] progress of the ghost plane below (this slab's
                         // memory, written by the neighbour below); null: Dirichlet plane
    int* ghost_hi;       // [R][tiles_j] ghost plane above; null: Dirichlet plane
    double* push_lo;     // the neighbour below's ghost plane above (its local plane nk+1)
    double* push_hi;     // the neighbour above's ghost plane below (its local plane 0)
    int* push_lo_flag;   // the neighbour below's ghost_hi
    int* push_hi_flag;   // the neighbour above's ghost_lo
    int lo_remote;       // the neighbour below / above runs on another GPU: its flags
    int hi_remote;       // and pushes are ordered at system scope (else GPU scope)
};
struct GsMaps {
    CUtensorMap ld[kGsMaxSlabs], st[kGsMaxSlabs];
};

struct GsParams {
    int ni, nj;
    int nslabs;
    int64_t pitch;         // row pitch of every slab grid (doubles)
    GsSlab slab[kGsMaxSlabs];
    int tiles_j, ntiles;
    int nch;               // column chunks per line (ceil((ni+2)/CW))
    long long tasks;       // sweeps * ntiles
    double b;
    int* ticket;           // atomic task counter
    int* prog;             // [R][ntiles] progress (encoded)
    int* err;              // error word (timeout): every role polls it and exits
    long long timeout;     // cycles without progress before a wait gives up
    int fault;             // test-only fault injection (sb_debug_fault), 0 = none
    const int2* order;     // ticket -> (sweep | slab << 16, J | K << 16), in wavefront order
    unsigned long long* prof;  // SB_GS_PROFILE builds: per-CTA cycle counters
};

template <int BJ_, int BK_, int CW_, int NS_, int LPT_>
struct GsCfg {
    static constexpr int BJ = BJ_, BK = BK_, CW = CW_, NS = NS_, LPT = LPT_;
    static_assert(BK % LPT == 0, "lines per thread must divide the tile's planes");
    static constexpr int NCOMP = BJ * BK / LPT;          // compute threads (LPT lines each:
                                                         // planes kl, kl + BK/LPT, ...)
    static_assert(NCOMP % 32 == 0, "whole compute warps");
    static constexpr int NT = NCOMP + 64;                // + loader warp + storer warp
    static constexpr int LJ = BJ + 2, LK = BK + 2;       // lines incl. halo
    static constexpr int LINES = LJ * LK;
    static constexpr int SLOT = CW * LINES;              // doubles per chunk slot
    static constexpr int SMAX = (BJ - 1) + (BK - 1);     // max line skew
    static constexpr int R = 8;                          // sweep slots for progress
    static constexpr int QS = NS + 4;                    // task queue entries (tasks may be
                                                         // as short as one chunk)
    static constexpr uint32_t BOX_BYTES = uint32_t(SLOT) * 8;
    // chunks in use at once: leading line's E chunk down to the trailing
    // line's chunk (the rest of the ring is prefetch)
    static_assert((NS - 2) * CW >= SMAX + 3, "too few chunk slots for the skew");
    static constexpr size_t SMEM_BYTES = size_t(NS) * SLOT * 8 + 24 * NS + 16 * QS + 64;
    // (full[NS], done[NS], empty[NS], task queue[QS], abort flag + spare)
};

struct GsTask {
    int s, J, K, tile, slab;  // s < 0: stop; K is slab-local
};

// progress encoding: (sweep+1) * (nch+1) + chunks_stored   (0 = nothing)
__device__ __forceinline__ int prog_val(int s, int chunks, int nch) { return (s + 1) * (nch + 1) + chunks; }

template <class C>
__device__ __forceinline__ bool prog_ready(const GsParams& p, int s, int tile, int need_chunks) {
    if (s < 0) return true;
    return ld_acquire(p.prog + (s % C::R) * p.ntiles + tile) >= prog_val(s, need_chunks, p.nch);
}

// Dependencies of one task, with the last progress value observed for each
// (a neighbour is usually several chunks ahead, so most checks hit the cache
// and the loader issues no global load at all).
struct GsDeps {
    const int* addr[6];
    int want_base[6];  // prog_val(sweep, 0, nch) of the awaited sweep
    int seen[6];
    int n;
    unsigned sys;      // bit k: entry k is a ghost flag written by another slab (system scope)
};

template <class C>
__device__ __forceinline__ void deps_init(const GsParams& p, const GsTask& t, GsDeps& d) {
    d.n = 0;
    d.sys = 0;
    auto add_at = [&](const int* a, int s) {
        d.addr[d.n] = a;
        d.want_base[d.n] = prog_val(s, 0, p.nch);
        d.seen[d.n] = 0;
        ++d.n;
    };
    auto add = [&](int s, int tile) { add_at(p.prog + (s % C::R) * p.ntiles + tile, s); };
    auto add_ghost = [&](const int* flags, int s, int remote) {
        if (remote) d.sys |= 1u << d.n;
        add_at(flags + (s % C::R) * p.tiles_j + t.J, s);
    };
    const GsSlab& S = p.slab[t.slab];
    if (t.s > 0) {
        add(t.s - 1, t.tile);
        if (t.J + 1 < p.tiles_j) add(t.s - 1, t.tile + 1);
        if (t.K + 1 < S.tiles_k) add(t.s - 1, t.tile + p.tiles_j);
        else if (S.ghost_hi) add_ghost(S.ghost_hi, t.s - 1, S.hi_remote);  // U: slab above, s-1
    }
    if (t.J > 0) add(t.s, t.tile - 1);
    if (t.K > 0) add(t.s, t.tile - p.tiles_j);
    else if (S.ghost_lo) add_ghost(S.ghost_lo, t.s, S.lo_remote);      // D: slab below, s
}

// true when chunk c of the task may be loaded; polls only stale entries
__device__ __forceinline__ bool deps_ready(GsDeps& d, int c) {
    bool ok = true;
    for (int k = 0; k < d.n; ++k) {
        const int want = d.want_base[k] + c + 1;
        if (d.seen[k] < want) {
            d.seen[k] = ((d.sys >> k) & 1) ? ld_acquire_sys(d.addr[k]) : ld_acquire(d.addr[k]);
            ok = ok && (d.seen[k] >= want);
        }
    }
    return ok;
}

template <class C>
__device__ __forceinline__ GsTask decode_task(const GsParams& p, long long tk) {
    GsTask t;
    if (tk >= p.tasks) {
        t.s = -1;
        t.J = t.K = t.tile = t.slab = 0;
        return t;
    }
    const int2 o = p.order[tk];
    t.s = o.x & 0xffff;
    t.slab = o.x >> 16;
    t.J = o.y & 0xffff;
    t.K = o.y >> 16;
    t.tile = p.slab[t.slab].tile0 + t.K * p.tiles_j + t.J;
    return t;
}

// Called in every polling loop.  Returns true when the launch is being
// abandoned: another thread flagged the error word, or this wait went
// p.timeout cycles without progress (it then flags it).  Every role then
// leaves its loops and the kernel exits normally, so the CUDA context stays
// usable and the host reads SB_ERR_TIMEOUT from the error word -- the GPU
// form of the reference's poisoned barriers (sync.py:31-32, team.py:42-64).
__device__ __forceinline__ bool gs_abort(const GsParams& p, long long t0) {
    if (*reinterpret_cast<volatile int*>(p.err)) return true;
    if (clock64() - t0 > p.timeout) {
        atomicExch(p.err, 1);
        __threadfence();
        return true;
    }
    __nanosleep(64);
    return false;
}

// A compute-side chunk wait: false when the launch is being abandoned.
__device__ __forceinline__ bool gs_wait(const GsParams& p, uint64_t* bar, uint32_t parity) {
    if (mbar_try_wait(bar, parity)) return true;
    const long long t0 = clock64();
    while (!mbar_try_wait(bar, parity))
        if (gs_abort(p, t0)) return false;
    return true;
}

// On abort the loader waits for its chunk loads still in flight (each is the
// latest load of its ring slot) to land before the CTA may exit.
template <class C>
__device__ void gs_loader_drain(uint64_t* full, uint32_t gload) {
    const uint32_t first = gload > uint32_t(C::NS) ? gload - C::NS : 0;
    for (uint32_t n = first; n < gload; ++n)
        while (!mbar_try_wait(&full[n % C::NS], (n / C::NS) & 1)) {
        }
}

// ---------------------------------------------------------------------------
// loader (one thread): dependency-checked chunk loads into free ring slots
template <class C>
__device__ void gs_loader(const GsMaps& maps, const GsParams& p, double* ring, uint64_t* full,
                          uint64_t* empty, GsTask* queue) {
    constexpr int NS = C::NS, CW = C::CW;
    const int nch = p.nch;
    uint32_t gload = 0;
    int lq = 0;
    long long t0 = clock64();
#ifdef SB_GS_PROFILE
    unsigned long long l_empty = 0, l_deps = 0;
#endif
    while (true) {
        const GsTask lt = decode_task<C>(p, atomicAdd(p.ticket, 1));
        queue[lq] = lt;  // published to the other warps by the next full[] phase
        lq = (lq + 1) % C::QS;
        const uint32_t slot0 = gload % NS;
        if (lt.s < 0) {
#ifdef SB_GS_PROFILE
            if (p.prof) {
                atomicAdd(&p.prof[4], l_empty);
                atomicAdd(&p.prof[5], l_deps);
            }
#endif
            // release the compute warps waiting for this (stop) task's first
            // chunk: complete that slot's barrier phase without data
            if (gload >= NS)
                while (!mbar_try_wait(&empty[slot0], ((gload - NS) / NS) & 1))
                    if (gs_abort(p, t0)) return gs_loader_drain<C>(full, gload);
            mbar_arrive(&full[slot0]);
            return;
        }
        GsDeps deps;
        deps_init<C>(p, lt, deps);
        for (int c = 0; c < nch; ++c, ++gload) {
            const uint32_t slot = gload % NS;
#ifdef SB_GS_PROFILE
            long long ta = clock64();
#endif
            if (gload >= NS) {  // the slot's previous chunk must have been stored
                while (!mbar_try_wait(&empty[slot], ((gload - NS) / NS) & 1))
                    if (gs_abort(p, t0)) return gs_loader_drain<C>(full, gload);
            }
#ifdef SB_GS_PROFILE
            long long tb = clock64();
            l_empty += tb - ta;
#endif
            while (!((c > 0 || prog_ready<C>(p, lt.s - (C::R - 1), lt.tile, nch)) && deps_ready(deps, c)))
                if (gs_abort(p, t0)) return gs_loader_drain<C>(full, gload);
#ifdef SB_GS_PROFILE
            l_deps += clock64() - tb;
#endif
            t0 = clock64();
            fence_proxy_async_global();
            mbar_arrive_expect_tx(&full[slot], C::BOX_BYTES);
            tma_load_3d(ring + size_t(slot) * C::SLOT, &maps.ld[lt.slab], c * CW, lt.J * C::BJ,
                        lt.K * C::BK, &full[slot]);
        }
    }
}

// storer (one thread): writes finished chunks back with TMA, frees the ring
// slot as soon as the store has read shared memory, and publishes progress
// once the data has landed in global memory
// Copies row block [J0, J0+BJ) x chunk c of one tile plane (a line set of
// a ring slot) into plane `dst` of a neighbour slab's grid (its ghost plane;
// peer memory when the neighbour is on another GPU): the interior rows, the
// chunk's columns inside the padded row.  One warp, 16-byte stores (the
// chunk's first column and the row pitch are even).
template <class C>
__device__ __forceinline__ void gs_push_plane(const GsParams& p, double* dst, const double* lines,
                                              int J0, int c, int lane) {
    constexpr int CW = C::CW, PAIRS = CW / 2;
    const int col0 = c * CW;
    const int ncol = min(CW, p.ni + 2 - col0);   // columns inside the padded row
    const int nrow = min(C::BJ, p.nj + 1 - J0);  // interior rows of the tile
    for (int idx = lane; idx < nrow * PAIRS; idx += 32) {
        const int jl = idx / PAIRS, x = 2 * (idx % PAIRS);
        if (x >= ncol) continue;
        const double* src = lines + jl * CW + x;
        double* out = dst + int64_t(J0 + jl) * p.pitch + col0 + x;
        if (x + 1 < ncol) *reinterpret_cast<double2*>(out) = make_double2(src[0], src[1]);
        else out[0] = src[0];
    }
}

// storer (one warp; lane 0 drives the TMA stores and the flags): writes
// finished chunks back with TMA, frees the ring slot as soon as the store has
// read shared memory, and publishes progress once the data has landed in
// global memory.  A tile holding a slab's edge plane also pushes that plane's
// chunk into the neighbour slab's ghost plane (the whole warp) and releases
// the neighbour's ghost flag.
template <class C>
__device__ void gs_storer(const GsMaps& maps, const GsParams& p, double* ring, uint64_t* done,
                          uint64_t* empty, uint64_t* full, GsTask* queue) {
    constexpr int NS = C::NS, CW = C::CW;
    const int nch = p.nch;
    const int lane = threadIdx.x & 31;
    uint32_t gstore = 0;
    int sq = 0;
    long long t0 = clock64();
    while (true) {
        // the task's first chunk being loaded implies its queue entry is written
        const uint32_t slot0 = gstore % NS;
        int ab = 0;
        GsTask t{};
        if (lane == 0) {
            while (!mbar_try_wait(&full[slot0], (gstore / NS) & 1))
                if (gs_abort(p, t0)) {
                    ab = 1;
                    break;
                }
            if (!ab) t = queue[sq];
        }
        if (__shfl_sync(0xffffffffu, ab, 0)) return;
        t.s = __shfl_sync(0xffffffffu, t.s, 0);
        t.J = __shfl_sync(0xffffffffu, t.J, 0);
        t.K = __shfl_sync(0xffffffffu, t.K, 0);
        t.tile = __shfl_sync(0xffffffffu, t.tile, 0);
        t.slab = __shfl_sync(0xffffffffu, t.slab, 0);
        sq = (sq + 1) % C::QS;
        if (t.s < 0) return;
        const GsSlab& S = p.slab[t.slab];
        const int J0 = 1 + t.J * C::BJ, K0 = 1 + t.K * C::BK;
        // owned planes of the tile: never store into the ghost plane above
        // (a partial top tile's halo line), which the neighbour writes
        const int nq = min(C::BK, S.nk + 1 - K0);
        const bool push_hi = S.push_hi && t.K == S.tiles_k - 1;
        const bool push_lo = S.push_lo && t.K == 0;
        int* flag = p.prog + (t.s % C::R) * p.ntiles + t.tile;
        for (int c = 0; c < nch; ++c, ++gstore) {
            const uint32_t slot = gstore % NS;
            const double* base = ring + size_t(slot) * C::SLOT;
            if (lane == 0) {
                while (!mbar_try_wait(&done[slot], (gstore / NS) & 1))
                    if (gs_abort(p, t0)) {
                        ab = 1;
                        break;
                    }
                if (!ab) {
                    t0 = clock64();
                    for (int q = 0; q < nq; ++q)
                        tma_store_3d(&maps.st[t.slab], base + ((q + 1) * C::LJ + 1) * CW, c * CW, J0,
                                     K0 + q);
                    bulk_commit();
                }
            }
            if (__shfl_sync(0xffffffffu, ab, 0)) return;
            if (push_hi)  // top owned plane -> the slab above's plane 0
                gs_push_plane<C>(p, S.push_hi, base + (nq * C::LJ + 1) * CW, J0, c, lane);
            if (push_lo)  // bottom plane -> the slab below's plane nk+1
                gs_push_plane<C>(p, S.push_lo, base + (C::LJ + 1) * CW, J0, c, lane);
            __syncwarp();  // the pushes have read the slot (and are ordered before lane 0's release)
            if (lane == 0) {
                bulk_wait_read<0>();  // the slot's data has left shared memory
                mbar_arrive(&empty[slot]);
                bulk_wait<0>();       // ... and landed in global memory
                fence_proxy_async_global();
                // test-only fault (sb_debug_fault(1)): tile 0 never publishes
                // sweep 0 past its first chunk, so its dependants time out
                if (p.fault == 1 && t.s == 0 && t.tile == 0 && c >= 1) continue;
                const int v = prog_val(t.s, c + 1, nch);
                st_release(flag, v);
                if (push_hi || push_lo) {
                    // the warp's pushes are ordered before these releases by the
                    // __syncwarp above (releases are cumulative); a peer GPU
                    // additionally needs the system-scope fence
                    const int gi = (t.s % C::R) * p.tiles_j + t.J;
                    if ((push_hi && S.hi_remote) || (push_lo && S.lo_remote)) __threadfence_system();
                    if (push_hi) {
                        if (S.hi_remote) st_release_sys(S.push_hi_flag + gi, v);
                        else st_release(S.push_hi_flag + gi, v);
                    }
                    if (push_lo) {
                        if (S.lo_remote) st_release_sys(S.push_lo_flag + gi, v);
                        else st_release(S.push_lo_flag + gi, v);
                    }
                }
            }
        }
    }
}

// One line of a tile as seen by its compute thread: column i at pi, column
// i+1 (the E neighbour) at pe in chunk ce, the start of chunk ce+1 at pnext.
struct GsLine {
    double* pi;
    double* pe;
    double* pnext;
    double wv;  // own previous value: the W neighbour
    int i, ce, line;
    bool in;    // inside the grid (partial tiles at the far edges)
};

template <class C>
__device__ __forceinline__ void gs_line_init(GsLine& L, double* smem, uint32_t gc, int jl, int kl,
                                             bool in) {
    constexpr int NS = C::NS, CW = C::CW;
    L.line = (kl + 1) * C::LJ + (jl + 1);
    L.i = 1 - (jl + kl);
    L.pi = smem + size_t(gc % NS) * C::SLOT + L.line * CW + max(L.i, 0);
    L.pe = L.pi + 1;
    L.ce = 0;
    L.pnext = smem + size_t((gc + 1) % NS) * C::SLOT + L.line * CW;
    L.wv = L.pi[-max(L.i, 0)];  // column 0: the Dirichlet halo (W of column 1)
    L.in = in;
}

// update column L.i (if active) and advance the line by one column
template <class C, bool INTERLEAVED, bool FULL>
__device__ __forceinline__ void gs_line_step(GsLine& L, double* smem, uint32_t gc, double b, int ni) {
    constexpr int NS = C::NS, CW = C::CW, LJ = C::LJ;
    const bool active = FULL || (L.in && (L.i >= 1) && (L.i <= ni));
    if (active) {
        const double e = *L.pe;
        const double sv = L.pi[-CW], nv = L.pi[CW];
        const double dv = L.pi[-LJ * CW], uv = L.pi[LJ * CW];
        double x;
        if (INTERLEAVED) {  // (ni >= 2 on this path: ni+2 is even)
            double tmp = __dadd_rn(e, sv);
            tmp = __dadd_rn(tmp, nv);
            tmp = __dadd_rn(tmp, dv);
            tmp = __dadd_rn(tmp, uv);
            x = __dmul_rn(b, __dadd_rn(L.wv, tmp));
        } else {
            double acc = __dadd_rn(L.wv, e);
            acc = __dadd_rn(acc, sv);
            acc = __dadd_rn(acc, nv);
            acc = __dadd_rn(acc, dv);
            acc = __dadd_rn(acc, uv);
            x = __dmul_rn(b, acc);
        }
        *L.pi = x;
        L.wv = x;
    }
    if (FULL || L.i >= 0) {  // advance: pi to column i+1, pe to column i+2
        L.pi = L.pe;
        if (((L.i + 2) & (CW - 1)) == 0) {
            ++L.ce;
            L.pe = L.pnext;
            L.pnext = smem + size_t((gc + L.ce + 1) % NS) * C::SLOT + L.line * CW;
        } else {
            ++L.pe;
        }
    }
    ++L.i;
}

// ---------------------------------------------------------------------------
template <class C, bool INTERLEAVED>
__global__ void __launch_bounds__(C::NT, 1)
gs_tile_kernel(const __grid_constant__ GsMaps maps, const __grid_constant__ GsParams p) {
    constexpr int BJ = C::BJ, CW = C::CW, NS = C::NS, SMAX = C::SMAX;
    extern __shared__ __align__(128) double smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + size_t(NS) * C::SLOT);
    uint64_t* done = full + NS;
    uint64_t* empty = done + NS;
    GsTask* queue = reinterpret_cast<GsTask*>(empty + NS);
    const int tid = threadIdx.x;

    if (tid == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&done[s], 1);
            mbar_init(&empty[s], 1);
        }
        *reinterpret_cast<volatile int*>(queue + C::QS) = 0;
        fence_mbar_init();
    }
    __syncthreads();

    if (tid >= C::NCOMP) {
        if (tid == C::NCOMP) {
            for (int i = 0; i < p.nslabs; ++i) tma_prefetch_desc(&maps.ld[i]);
            gs_loader<C>(maps, p, smem, full, empty, queue);
        } else if (tid >= C::NCOMP + 32) {  // the storer warp
            if (tid == C::NCOMP + 32)
                for (int i = 0; i < p.nslabs; ++i) tma_prefetch_desc(&maps.st[i]);
            gs_storer<C>(maps, p, smem, done, empty, full, queue);
        }
        return;
    }

    // compute thread: LPT lines of the tile.  All chunk waits and releases
    // are CTA-uniform events (functions of the step only), handled by thread 0
    // around the per-step named barrier: when the trailing line completes a
    // chunk, every thread fences its shared-memory writes for the async proxy
    // and after the barrier thread 0 hands the chunk to the storer.
    constexpr int LPT = C::LPT, KSTEP = C::BK / C::LPT;
    // abort flag: thread 0 sets it when a chunk wait gives up (gs_abort); the
    // other compute threads read it after the step barrier that follows
    volatile int* abort_s = reinterpret_cast<volatile int*>(queue + C::QS);
    const int jl = tid % BJ, kl0 = tid / BJ;
    const double b = p.b;
    const int nch = p.nch, ni = p.ni;
    const int nsteps = ni + SMAX;
    uint32_t gc = 0;  // global chunk index of the current task's chunk 0
    int q = 0;
#ifdef SB_GS_PROFILE
    unsigned long long w_start = 0, w_chunk = 0, n_tasks = 0;
    const long long k_t0 = clock64();
#endif
    while (true) {
#ifdef SB_GS_PROFILE
        long long tw = clock64();
#endif
        if (tid == 0 && !gs_wait(p, &full[gc % NS], (gc / NS) & 1))  // chunk 0 (+ queue entry)
            *abort_s = 1;
#ifdef SB_GS_PROFILE
        w_start += clock64() - tw;
        ++n_tasks;
#endif
        named_bar_sync(1, C::NCOMP);
        if (*abort_s) break;
        const GsTask t = queue[q];
        q = (q + 1) % C::QS;
        if (t.s < 0) break;
        const int J0 = 1 + t.J * BJ, K0 = 1 + t.K * C::BK;
        const int nk = p.slab[t.slab].nk;
        GsLine lines[LPT];
#pragma unroll
        for (int l = 0; l < LPT; ++l) {
            const int kl = kl0 + l * KSTEP;
            gs_line_init<C>(lines[l], smem, gc, jl, kl, (J0 + jl <= p.nj) && (K0 + kl <= nk));
        }
        int ready = 1;               // chunks known loaded (thread 0)
        int completed = 0;           // chunks completed so far
        int released = 0;            // chunks handed to the storer (thread 0)
        constexpr int POS_LEAD = CW - 3;                        // (st+3) % CW == 0
        constexpr int POS_FIN = ((SMAX - 2) % CW + CW) % CW;    // (st+2-SMAX) % CW == 0
        // One block of CW plane steps.  FULL: every line computes at every step
        // of the block (no prologue/epilogue of the skew, no partial tile).
        // Returns true when the launch is being abandoned (gs_abort).
        auto block = [&](const int st0, auto full_tag) -> bool {
            constexpr bool FULL = decltype(full_tag)::value;
#pragma unroll
            for (int pos = 0; pos < CW; ++pos) {
                const int st = st0 + pos;
                if (pos == POS_FIN + 1 || pos == 0) {  // every thread fenced before the last barrier
                    if (tid == 0)
                        while (released < completed) mbar_arrive(&done[(gc + released++) % NS]);
                }
#pragma unroll
                for (int l = 0; l < LPT; ++l) gs_line_step<C, INTERLEAVED, FULL>(lines[l], smem, gc, b, ni);
                if (pos == POS_FIN || (!FULL && st == nsteps - 1)) {
                    const int fin = (st >= nsteps - 1) ? nch : min(nch, max(0, (st + 2 - SMAX) / CW));
                    if (fin > completed) {
                        fence_proxy_async_smem();  // this thread's smem writes -> async proxy
                        completed = fin;           // released after this step's barrier
                    }
                }
                if (pos == POS_LEAD && tid == 0) {  // the leading line reads column st+3 next step
                    const int cneed = (st + 3) / CW;
                    if (cneed < nch && cneed >= ready) {
#ifdef SB_GS_PROFILE
                        long long tc = clock64();
#endif
                        if (!gs_wait(p, &full[(gc + cneed) % NS], ((gc + cneed) / NS) & 1))
                            *abort_s = 1;
#ifdef SB_GS_PROFILE
                        w_chunk += clock64() - tc;
#endif
                        ready = cneed + 1;
                    }
                }
                named_bar_sync(1, C::NCOMP);
                if (pos == POS_LEAD && *abort_s) return true;
                if (!FULL && st == nsteps - 1) break;
            }
            return false;
        };
        // full blocks: the trailing line (skew SMAX) is at column >= 1 at the
        // block's first step and the leading line at column <= ni at its last
        const bool tile_full = (J0 + C::BJ - 1 <= p.nj) && (K0 + C::BK - 1 <= nk);
        bool aborted = false;
        for (int st0 = 0; st0 < nsteps && !aborted; st0 += CW) {
            if (tile_full && st0 + 1 - SMAX >= 1 && st0 + CW <= ni && st0 + CW < nsteps)
                aborted = block(st0, std::true_type{});
            else
                aborted = block(st0, std::false_type{});
        }
        if (aborted) break;
        if (tid == 0) {
            while (released < completed) mbar_arrive(&done[(gc + released++) % NS]);
        }
        gc += nch;
    }
#ifdef SB_GS_PROFILE
    if (tid == 0 && p.prof) {
        atomicAdd(&p.prof[0], (unsigned long long)(clock64() - k_t0));
        atomicAdd(&p.prof[1], w_start);
        atomicAdd(&p.prof[2], w_chunk);
        atomicAdd(&p.prof[3], n_tasks);
    }
#endif
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
// 16 x 6-line tiles with 4-slot rings: 74 KB of shared memory, three CTAs per
// SM.  The resident CTAs hide each other's chunk waits and barriers (one
// 16 x 16 CTA per SM, 5 slots: 239.5 GLUP/s at 512^3 x 100; 16 x 8, two per
// SM: 245.7; 16 x 6, three per SM: 248.8; 16 x 4, four: 236.4; 8 x 12: 237).
using GsC = GsCfg<16, 6, 16, 4, 1>;
using GsC1 = GsCfg<16, 16, 16, 5, 1>;  // one CTA per SM (SB_GSCFG=1)

// Per-device launch state (ticket/error words, progress flags, order table).
// Launches on one device that use it are serialised whatever their stream:
// each waits for `last` (recorded after the previous launch) and host-side
// updates happen under `mu`, so concurrent sb_gs calls on two streams of one
// device never share the counters of a running kernel.
struct GsScratch {
    std::mutex mu;
    int* words = nullptr;  // ticket, err
    int* prog = nullptr;
    size_t prog_cap = 0;
    int2* order = nullptr;
    size_t order_cap = 0;
    std::vector<int> key;  // what the uploaded order table describes
    cudaEvent_t last = nullptr;
};
static GsScratch g_gs[16];

// Test-only fault injection (sb_debug_fault): applies to later launches.
static int g_fault = 0;
static long long g_timeout = 1LL << 35;  // ~17 s at 1.9 GHz without progress
#ifdef SB_GS_PROFILE
static unsigned long long* g_gs_prof = nullptr;
extern "C" void sb_gs_profile(unsigned long long* out) {
    cudaDeviceSynchronize();
    if (g_gs_prof) cudaMemcpy(out, g_gs_prof, 6 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
}
#endif

// Ticket order over `sweeps` sweeps of the tiles of one launch, in windows
// of `window` sweeps: inside a window by tau = (J + K) + 2 * sweep, then
// sweep, then J; windows one after another.  K is the tile's global K index
// over all slabs of the grid (kt[g] = K tiles of slab g, in z order); only
// tiles of slabs in this launch (mine[g] >= 0: its index in the launch) get
// tickets.  Every dependency of task (s, J, K) -- (s, J-1, K), (s, J, K-1)
// at tau-1, (s-1, J+1, K), (s-1, J, K+1) at tau-1, (s-1, J, K) at tau-2,
// (s-R+1, J, K) at tau-2(R-1), or an earlier window -- has a smaller
// (window, tau) key, in this launch or in another GPU's launch of the same
// order: every device takes its tasks in key order, so the task with the
// smallest unfinished key anywhere is always running -- no deadlock, on one
// persistent grid or across GPUs.  Successive sweeps advance together in a
// diagonal band (the paper's multi-wavefront GS); the window bounds how many
// are in flight, so that a tile's next sweep reads its previous sweep's data
// while it is still in L2.
static std::vector<int2> wavefront_order(int tiles_j, const std::vector<int>& kt,
                                         const std::vector<int>& mine, int sweeps, int window) {
    std::vector<int> kslab, klocal;  // global K -> (slab, local K)
    for (size_t g = 0; g < kt.size(); ++g)
        for (int k = 0; k < kt[g]; ++k) {
            kslab.push_back((int)g);
            klocal.push_back(k);
        }
    const int tiles_k = (int)kslab.size();
    std::vector<int2> ord;
    const int dmax = tiles_j + tiles_k - 2;
    for (int s0 = 0; s0 < sweeps; s0 += window) {
        const int ns = std::min(window, sweeps - s0);
        for (int tau = 0; tau <= dmax + 2 * (ns - 1); ++tau)
            for (int s = std::max(0, (tau - dmax + 1) / 2); s < ns && 2 * s <= tau; ++s) {
                const int d = tau - 2 * s;
                if (d > dmax) continue;
                for (int J = std::max(0, d - (tiles_k - 1)); J < tiles_j && J <= d; ++J) {
                    const int Kg = d - J, g = kslab[Kg];
                    if (mine[g] >= 0)
                        ord.push_back(make_int2((s0 + s) | (mine[g] << 16), J | (klocal[Kg] << 16)));
                }
            }
    }
    return ord;
}

static int gs_window() {
    static int w = tune_env("SB_GS_WINDOW") ? std::max(1, atoi(tune_env("SB_GS_WINDOW"))) : 3;
    return w;
}

// Host view of one slab of a launch (a single-grid call is one slab without
// neighbours).
struct GsLaunchSlab {
    double* grid = nullptr;
    int nk = 0;
    int* ghost_lo = nullptr;
    int* ghost_hi = nullptr;
    double* push_lo = nullptr;
    double* push_hi = nullptr;
    int* push_lo_flag = nullptr;
    int* push_hi_flag = nullptr;
    int lo_remote = 0, hi_remote = 0;  // neighbour on another device
};

// Sweeps per launch: bounded by the order table size and the int32
// progress encoding.
template <class C>
static int64_t gs_batch_limit(int ni, int64_t ntiles) {
    const int64_t nch64 = (ni + 2 + C::CW - 1) / C::CW;
    return std::max<int64_t>(1, std::min<int64_t>(
        std::min<int64_t>(512, ((int64_t(1) << 30) / (nch64 + 1)) - 2), (int64_t(1) << 26) / ntiles));
}

// Launches `iters` sweeps of the slabs sl[0..nsl) (all on the current
// device; kt / mine: K tiles of every slab of the global grid and the
// launch index of each, see wavefront_order) in batches of at most
// gs_batch_limit sweeps.  reset_ghosts: zero the slabs' ghost flags before
// each batch on `st` (when every neighbour is in this launch); cross-GPU
// callers reset them themselves and pass one batch at a time.
template <class C>
static int gs_launch_slabs(const GsLaunchSlab* sl, int nsl, const std::vector<int>& kt,
                           const std::vector<int>& mine, int ni, int nj, int64_t iters, double b,
                           bool inter, cudaStream_t st, int64_t pitch, int window, bool reset_ghosts) {
    int dev;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    if (dev >= 16) return fail(SB_ERR_CUDA, "device index %d unsupported", dev);
    if (nsl < 1 || nsl > kGsMaxSlabs) return fail(SB_ERR_ARGUMENT, "%d slabs in one launch", nsl);
    GsScratch& S = g_gs[dev];
    std::lock_guard<std::mutex> lk(S.mu);
    int* counters;
    int sms;
    int rc = get_counters(&counters, &sms);
    if (rc) return rc;
    if (!S.last && (e = cudaEventCreateWithFlags(&S.last, cudaEventDisableTiming)) != cudaSuccess)
        return cuda_fail(e, "cudaEventCreate");
    // the previous launch on this device (any stream) has finished with the scratch
    if ((e = cudaStreamWaitEvent(st, S.last, 0)) != cudaSuccess) return cuda_fail(e, "cudaStreamWaitEvent");

    const int tiles_j = (nj + C::BJ - 1) / C::BJ;
    int ntiles = 0;
    for (int i = 0; i < nsl; ++i) {
        const int tk = (sl[i].nk + C::BK - 1) / C::BK;
        if (tiles_j > 32767 || tk > 32767) return fail(SB_ERR_DIMENSION, "grid too large for GS tiling");
        ntiles += tiles_j * tk;
    }
    if (!S.words && (e = cudaMalloc(&S.words, 64 * sizeof(int))) != cudaSuccess)
        return cuda_fail(e, "cudaMalloc");
    const size_t need = size_t(C::R) * ntiles;
    if (S.prog_cap < need) {
        if (S.prog) cudaFree(S.prog);
        if ((e = cudaMalloc(&S.prog, need * sizeof(int))) != cudaSuccess) return cuda_fail(e, "cudaMalloc");
        S.prog_cap = need;
    }
    const int batch = (int)std::min<int64_t>(iters, gs_batch_limit<C>(ni, ntiles));
    auto upload_order = [&](int n) -> int {
        std::vector<int> key = {tiles_j, window, n, C::BJ, C::BK};
        key.insert(key.end(), kt.begin(), kt.end());
        key.insert(key.end(), mine.begin(), mine.end());
        if (key == S.key) return SB_OK;
        const std::vector<int2> ord = wavefront_order(tiles_j, kt, mine, n, window);
        if (S.order_cap < ord.size()) {
            if (S.order) cudaFree(S.order);
            S.order = nullptr;
            if ((e = cudaMalloc(&S.order, ord.size() * sizeof(int2))) != cudaSuccess)
                return cuda_fail(e, "cudaMalloc(order)");
            S.order_cap = ord.size();
        }
        // stream-ordered: a previous launch on this stream may still read the table
        if ((e = cudaMemcpyAsync(S.order, ord.data(), ord.size() * sizeof(int2), cudaMemcpyHostToDevice,
                                 st)) != cudaSuccess)
            return cuda_fail(e, "cudaMemcpy(order)");
        if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return cuda_fail(e, "order upload");
        S.key = key;
        return SB_OK;
    };

    GsMaps maps;
    GsParams p;
    memset(&p, 0, sizeof p);
    const int64_t nip = ni + 2, njp = nj + 2;
    if (pitch <= 0) pitch = nip;
    int tile0 = 0;
    for (int i = 0; i < nsl; ++i) {
        if ((rc = make_grid_map3p(&maps.ld[i], sl[i].grid, nip, njp, sl[i].nk + 2, C::CW, C::LJ, C::LK,
                                  pitch)) ||
            (rc = make_grid_map3p(&maps.st[i], sl[i].grid, nip, njp, sl[i].nk + 2, C::CW, C::BJ, 1, pitch)))
            return rc;
        GsSlab& X = p.slab[i];
        X.nk = sl[i].nk;
        X.tiles_k = (sl[i].nk + C::BK - 1) / C::BK;
        X.tile0 = tile0;
        tile0 += X.tiles_k * tiles_j;
        X.ghost_lo = sl[i].ghost_lo;
        X.ghost_hi = sl[i].ghost_hi;
        X.push_lo = sl[i].push_lo;
        X.push_hi = sl[i].push_hi;
        X.push_lo_flag = sl[i].push_lo_flag;
        X.push_hi_flag = sl[i].push_hi_flag;
        X.lo_remote = sl[i].lo_remote;
        X.hi_remote = sl[i].hi_remote;
    }

    auto kern_n = gs_tile_kernel<C, false>;
    auto kern_i = gs_tile_kernel<C, true>;
    int occ = 0;
    if ((rc = ctas_per_sm((const void*)kern_i, C::NT, C::SMEM_BYTES, &occ)) ||
        (rc = ctas_per_sm((const void*)kern_n, C::NT, C::SMEM_BYTES, &occ)))
        return rc;
    p.ni = ni;
    p.nj = nj;
    p.nslabs = nsl;
    p.pitch = pitch;
    p.tiles_j = tiles_j;
    p.ntiles = ntiles;
    p.nch = (ni + 2 + C::CW - 1) / C::CW;
    p.b = b;
    p.ticket = S.words;
    p.err = S.words + 1;
    p.timeout = g_timeout;
    p.fault = g_fault;
    p.prog = S.prog;
    p.prof = nullptr;
#ifdef SB_GS_PROFILE
    static unsigned long long* prof = nullptr;
    if (!prof) cudaMalloc(&prof, 64);
    cudaMemsetAsync(prof, 0, 64, st);
    p.prof = prof;
    g_gs_prof = prof;
#endif
    const size_t gbytes = size_t(C::R) * tiles_j * sizeof(int);
    for (int64_t done = 0; done < iters;) {
        const int n = (int)std::min<int64_t>(iters - done, batch);
        if ((rc = upload_order(n))) return rc;
        p.order = S.order;
        p.tasks = (long long)n * ntiles;
        if ((e = cudaMemsetAsync(S.words, 0, 64 * sizeof(int), st)) != cudaSuccess)
            return cuda_fail(e, "memset");
        if ((e = cudaMemsetAsync(S.prog, 0, need * sizeof(int), st)) != cudaSuccess)
            return cuda_fail(e, "memset");
        if (reset_ghosts)
            for (int i = 0; i < nsl; ++i)
                for (int* gf : {sl[i].ghost_lo, sl[i].ghost_hi})
                    if (gf && (e = cudaMemsetAsync(gf, 0, gbytes, st)) != cudaSuccess)
                        return cuda_fail(e, "memset(ghost flags)");
        const int grid_ctas = (int)std::min<long long>((long long)sms * occ, p.tasks);
        if (inter) kern_i<<<grid_ctas, C::NT, C::SMEM_BYTES, st>>>(maps, p);
        else kern_n<<<grid_ctas, C::NT, C::SMEM_BYTES, st>>>(maps, p);
        if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "gs launch");
        if ((e = cudaEventRecord(S.last, st)) != cudaSuccess) return cuda_fail(e, "cudaEventRecord");
        done += n;
    }
    return SB_OK;
}

// One grid (sb_gs): a launch of one slab without neighbours.
template <class C>
static int gs_launch(double* grid, int ni, int nj, int nk, int64_t iters, double b, bool inter,
                     cudaStream_t st, int64_t pitch = 0) {
    GsLaunchSlab one;
    one.grid = grid;
    one.nk = nk;
    return gs_launch_slabs<C>(&one, 1, {(nk + C::BK - 1) / C::BK}, {0}, ni, nj, iters, b, inter, st,
                              pitch, gs_window(), false);
}

int gs_serial_run(double* grid, int ni, int nj, int nk, int64_t iters, double b, int kernel,
                  cudaStream_t st);

// Grids TMA cannot describe directly (odd ni: the row pitch (ni+2)*8 bytes is
// not a multiple of 16; or a base address that is not 16-byte aligned) run
// the tile kernel on a pitched copy: rows padded to an even number of doubles
// (the extra column lies outside the tensor map, so it is never read or
// written), copied in and out with cudaMemcpy2D.  One scratch buffer per
// device, grown on demand, stream-ordered like the rest of sb_gs.
struct GsPitched {
    std::mutex mu;
    double* buf = nullptr;
    size_t cap = 0;  // doubles
    cudaEvent_t last = nullptr;  // after the previous user's copy-out (any stream)
};
static GsPitched g_gs_pitched[16];

// frees the pitched-copy buffer of `dev` (caller synchronised the device);
// true if there was one
bool gs_release(int dev) {
    if (dev < 0 || dev >= 16) return false;
    GsPitched& P = g_gs_pitched[dev];
    std::lock_guard<std::mutex> lk(P.mu);
    const bool had = P.buf != nullptr;
    if (P.buf) cudaFree(P.buf);
    P.buf = nullptr;
    P.cap = 0;
    return had;
}

// true if `dev` holds buffers that sb_release_caches would free
bool gs_holds(int dev) {
    if (dev < 0 || dev >= 16) return false;
    std::lock_guard<std::mutex> lk(g_gs_pitched[dev].mu);
    return g_gs_pitched[dev].buf != nullptr;
}

static int gs_run_pitched(double* grid, int ni, int nj, int nk, int64_t iters, double b,
                          bool inter, cudaStream_t st) {
    int dev;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    if (dev >= 16) return fail(SB_ERR_CUDA, "device index %d unsupported", dev);
    GsPitched& P = g_gs_pitched[dev];
    std::lock_guard<std::mutex> lk(P.mu);
    if (!P.last && (e = cudaEventCreateWithFlags(&P.last, cudaEventDisableTiming)) != cudaSuccess)
        return cuda_fail(e, "cudaEventCreate");
    if ((e = cudaStreamWaitEvent(st, P.last, 0)) != cudaSuccess) return cuda_fail(e, "cudaStreamWaitEvent");
    const int64_t nip = ni + 2, pitch = (nip + 1) / 2 * 2, rows = int64_t(nj + 2) * (nk + 2);
    const size_t need = size_t(pitch) * size_t(rows);
    if (P.cap < need) {
        if (P.buf && (e = cudaStreamSynchronize(st)) != cudaSuccess) return cuda_fail(e, "sync");
        if (P.buf) cudaFree(P.buf);
        P.buf = nullptr;
        P.cap = 0;
        if ((e = cudaMalloc(&P.buf, need * sizeof(double))) != cudaSuccess)
            return cuda_fail(e, "cudaMalloc(pitched GS grid)");
        P.cap = need;
    }
    if ((e = cudaMemcpy2DAsync(P.buf, pitch * 8, grid, nip * 8, nip * 8, rows,
                               cudaMemcpyDeviceToDevice, st)) != cudaSuccess)
        return cuda_fail(e, "cudaMemcpy2DAsync(in)");
    int rc = (iters <= 2)
                 ? gs_launch<GsC1>(P.buf, ni, nj, nk, iters, b, inter, st, pitch)
                 : gs_launch<GsC>(P.buf, ni, nj, nk, iters, b, inter, st, pitch);
    if (rc) return rc;
    if ((e = cudaMemcpy2DAsync(grid, nip * 8, P.buf, pitch * 8, nip * 8, rows,
                               cudaMemcpyDeviceToDevice, st)) != cudaSuccess)
        return cuda_fail(e, "cudaMemcpy2DAsync(out)");
    if ((e = cudaEventRecord(P.last, st)) != cudaSuccess) return cuda_fail(e, "cudaEventRecord");
    return SB_OK;
}

int gs_run(double* grid, int ni, int nj, int nk, int64_t iters, double b, int kernel,
           cudaStream_t st) {
    if (!tma_ok(grid, ni)) {
        // tiny grids: the exact serial kernel is cheaper than the copies
        if (int64_t(ni) * nj * nk * iters < (int64_t(1) << 16))
            return gs_serial_run(grid, ni, nj, nk, iters, b, kernel, st);
        // ni < 2: the interleaved association degenerates to the naive one
        // (reference kernels.py:168-176)
        return gs_run_pitched(grid, ni, nj, nk, iters, b,
                              kernel == SB_KERNEL_GS_INTERLEAVED && ni >= 2, st);
    }
    static const int v = tune_env("SB_GSCFG") ? atoi(tune_env("SB_GSCFG")) : 0;  // tuning
    const bool inter = kernel == SB_KERNEL_GS_INTERLEAVED;
    // one or two sweeps per call (the GS z-pipeline's stages): the 16 x 16
    // tiles' shorter tile-wavefront fill wins (512^3: 1 sweep 0.90 vs 1.31 ms,
    // 2 sweeps 1.33 vs 1.44); from 4 sweeps on, the 16 x 6 tiles
    if (v == 1 || (v == 0 && iters <= 2))
        return gs_launch<GsC1>(grid, ni, nj, nk, iters, b, inter, st);
    return gs_launch<GsC>(grid, ni, nj, nk, iters, b, inter, st);
}

// The cross-GPU z-pipeline in one persistent launch per device
// (sb_gs_slabs): slab g (grids[g] on devices[g], local planes 0 and nk_g+1
// are ghost planes) pushes its edge planes' chunks into its neighbours'
// ghost planes as it stores them and releases their ghost flags, so sweep s
// of slab g runs behind slab g-1's sweep s and slab g+1's sweep s-1 at chunk
// granularity (wavefront_order keys are global, so the launches cannot
// deadlock).  Slabs sharing a device form one launch on streams[first of
// them].  Returns SB_ERR_PLAN when the layout is not eligible (odd ni,
// unaligned grids, more than kGsMaxSlabs slabs on one device): the caller
// then runs the launch-per-sweep pipeline.
int gs_slabs_fused(int nslabs, const int* devices, double* const* grids, const int64_t* nks, int ni,
                   int nj, int64_t iters, double b, int kernel, void* const* streams) {
    using C = GsC;
    if (ni % 2) return SB_ERR_PLAN;
    for (int g = 0; g < nslabs; ++g)
        if (!tma_ok(grids[g], ni)) return SB_ERR_PLAN;
    // launch groups: slabs per device, in z order
    std::vector<int> devs;
    std::vector<std::vector<int>> members;
    for (int g = 0; g < nslabs; ++g) {
        auto it = std::find(devs.begin(), devs.end(), devices[g]);
        if (it == devs.end()) {
            devs.push_back(devices[g]);
            members.push_back({g});
        } else {
            members[it - devs.begin()].push_back(g);
        }
    }
    for (auto& m : members)
        if ((int)m.size() > kGsMaxSlabs) return SB_ERR_PLAN;
    // the storer warps push into the neighbours' memory: neighbouring slabs on
    // different GPUs need peer access (else the launch-per-sweep pipeline,
    // whose ghost copies go through cudaMemcpyPeerAsync, runs)
    for (int g = 0; g + 1 < nslabs; ++g)
        if (!peer_reachable(devices[g], devices[g + 1])) return SB_ERR_PLAN;
    const int tiles_j = (nj + C::BJ - 1) / C::BJ;
    const size_t gbytes = size_t(C::R) * tiles_j * sizeof(int);
    std::vector<int> kt(nslabs);
    for (int g = 0; g < nslabs; ++g) kt[g] = int((nks[g] + C::BK - 1) / C::BK);
    // ghost flags: [R][tiles_j] per inner side, in the slab's own memory
    std::vector<int*> glo(nslabs, nullptr), ghi(nslabs, nullptr);
    cudaError_t e = cudaSuccess;
    int rc = SB_OK;
    auto release = [&]() {
        for (int g = 0; g < nslabs; ++g) {
            cudaSetDevice(devices[g]);
            if (glo[g]) cudaFree(glo[g]);
            if (ghi[g]) cudaFree(ghi[g]);
        }
    };
    for (int g = 0; g < nslabs && rc == SB_OK; ++g) {
        if ((e = cudaSetDevice(devices[g])) != cudaSuccess) rc = cuda_fail(e, "cudaSetDevice");
        else if (g > 0 && (e = cudaMalloc(&glo[g], gbytes)) != cudaSuccess) rc = cuda_fail(e, "cudaMalloc");
        else if (g + 1 < nslabs && (e = cudaMalloc(&ghi[g], gbytes)) != cudaSuccess)
            rc = cuda_fail(e, "cudaMalloc");
    }
    if (rc) {
        release();
        return rc;
    }
    const int64_t plane = int64_t(ni + 2) * (nj + 2);
    std::vector<std::vector<GsLaunchSlab>> ls(devs.size());
    std::vector<std::vector<int>> mine(devs.size(), std::vector<int>(nslabs, -1));
    for (size_t d = 0; d < devs.size(); ++d)
        for (size_t i = 0; i < members[d].size(); ++i) {
            const int g = members[d][i];
            GsLaunchSlab x;
            x.grid = grids[g];
            x.nk = int(nks[g]);
            x.ghost_lo = glo[g];
            x.ghost_hi = ghi[g];
            if (g > 0) {
                x.push_lo = grids[g - 1] + (nks[g - 1] + 1) * plane;  // below: its plane nk+1
                x.push_lo_flag = ghi[g - 1];
                x.lo_remote = devices[g - 1] != devices[g];
            }
            if (g + 1 < nslabs) {
                x.push_hi = grids[g + 1];  // above: its plane 0
                x.push_hi_flag = glo[g + 1];
                x.hi_remote = devices[g + 1] != devices[g];
            }
            ls[d].push_back(x);
            mine[d][g] = int(i);
        }
    const bool inter = kernel == SB_KERNEL_GS_INTERLEAVED;
    // one device: one launch, the single-grid schedule; several: a wider
    // sweep window so that every GPU of the pipeline has work in flight
    const int window = devs.size() == 1 ? gs_window() : gs_window() * int(devs.size());
    auto stream_of = [&](size_t d) { return static_cast<cudaStream_t>(streams[members[d][0]]); };
    if (devs.size() == 1) {
        cudaSetDevice(devs[0]);
        rc = gs_launch_slabs<C>(ls[0].data(), (int)ls[0].size(), kt, mine[0], ni, nj, iters, b, inter,
                                stream_of(0), 0, window, true);
        if (rc == SB_OK && (e = cudaStreamSynchronize(stream_of(0))) != cudaSuccess)
            rc = cuda_fail(e, "slab sweeps");
        if (rc == SB_OK) rc = gs_check_error(stream_of(0));
    } else {
        int64_t ntiles_max = 0;
        for (size_t d = 0; d < devs.size(); ++d) {
            int64_t n = 0;
            for (int g : members[d]) n += int64_t(kt[g]) * tiles_j;
            ntiles_max = std::max(ntiles_max, n);
        }
        const int64_t batch = gs_batch_limit<C>(ni, ntiles_max);
        for (int64_t done = 0; done < iters && rc == SB_OK;) {
            const int64_t n = std::min(batch, iters - done);
            // every device's ghost flags are zero before any launch of the batch starts
            for (size_t d = 0; d < devs.size() && rc == SB_OK; ++d) {
                cudaSetDevice(devs[d]);
                for (int g : members[d])
                    for (int* gf : {glo[g], ghi[g]})
                        if (gf && (e = cudaMemsetAsync(gf, 0, gbytes, stream_of(d))) != cudaSuccess)
                            rc = cuda_fail(e, "memset(ghost flags)");
            }
            for (size_t d = 0; d < devs.size() && rc == SB_OK; ++d) {
                cudaSetDevice(devs[d]);
                if ((e = cudaStreamSynchronize(stream_of(d))) != cudaSuccess) rc = cuda_fail(e, "sync");
            }
            for (size_t d = 0; d < devs.size() && rc == SB_OK; ++d) {
                cudaSetDevice(devs[d]);
                rc = gs_launch_slabs<C>(ls[d].data(), (int)ls[d].size(), kt, mine[d], ni, nj, n, b, inter,
                                        stream_of(d), 0, window, false);
            }
            for (size_t d = 0; d < devs.size(); ++d) {  // all launches end before the next batch
                cudaSetDevice(devs[d]);
                if ((e = cudaStreamSynchronize(stream_of(d))) != cudaSuccess && rc == SB_OK)
                    rc = cuda_fail(e, "slab sweeps");
                if (rc == SB_OK) rc = gs_check_error(stream_of(d));
            }
            done += n;
        }
    }
    release();
    return rc;
}

int gs_serial_run(double* grid, int ni, int nj, int nk, int64_t iters, double b, int kernel,
                  cudaStream_t st) {
    const bool inter = (kernel == SB_KERNEL_GS_INTERLEAVED);
    for (int64_t done = 0; done < iters;) {
        const int n = (int)std::min<int64_t>(iters - done, 1 << 20);
        if (inter) gs_serial_kernel<true><<<1, 32, 0, st>>>(grid, ni, nj, nk, n, b);
        else gs_serial_kernel<false><<<1, 32, 0, st>>>(grid, ni, nj, nk, n, b);
        done += n;
    }
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? SB_OK : cuda_fail(e, "gs_serial launch");
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

extern "C" int sb_debug_fault(int kind, int64_t timeout_cycles) {
    using namespace sb;
    clear_error();
    if (kind < 0 || kind > 1) return fail(SB_ERR_ARGUMENT, "unknown fault kind %d", kind);
    g_fault = kind;
    g_timeout = timeout_cycles > 0 ? timeout_cycles : (1LL << 35);
    return SB_OK;
}

extern "C" int sb_sync(void* stream) {
    using namespace sb;
    clear_error();
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "stream synchronize");
    return gs_check_error(st);
}

// The library's "serial engine": straightforward kernels with none of the
// tiling, pipelining or temporal blocking -- one plain sweep per launch for
// Jacobi, a single thread in exact lexicographic order for GS.  The CLI's
// verify compares the optimised paths against it (reference cli.py:297-331
// compares its parallel variants against run_serial the same way).
extern "C" int sb_reference_sweeps(int kernel, double* grid, double* scratch, int64_t ni, int64_t nj,
                                   int64_t nk, int64_t iters, double a, double b, void* stream,
                                   int* result_in_scratch) {
    using namespace sb;
    clear_error();
    int rc = check_dims(ni, nj, nk);
    if (rc) return rc;
    if (iters < 0) return fail(SB_ERR_PLAN, "iter_end must be >= 0, got %lld", (long long)iters);
    if (!grid || !result_in_scratch) return fail(SB_ERR_ARGUMENT, "null pointer");
    *result_in_scratch = 0;
    if (iters == 0) return SB_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (kernel == SB_KERNEL_JACOBI) {
        if (!scratch || scratch == grid) return fail(SB_ERR_ARGUMENT, "Jacobi needs a distinct scratch grid");
        if ((rc = halo_copy(grid, scratch, (int)ni, (int)nj, (int)nk, st))) return rc;
        double* src = grid;
        double* dst = scratch;
        for (int64_t s = 0; s < iters; ++s) {
            if ((rc = jacobi_generic_sweep(src, dst, (int)ni, (int)nj, (int)nk, a, b, st))) return rc;
            std::swap(src, dst);
        }
        *result_in_scratch = (src == scratch);
        return SB_OK;
    }
    if (kernel != SB_KERNEL_GS_NAIVE && kernel != SB_KERNEL_GS_INTERLEAVED)
        return fail(SB_ERR_PLAN, "unknown kernel %d", kernel);
    return gs_serial_run(grid, (int)ni, (int)nj, (int)nk, iters, b, kernel, st);
}

// One line update (reference kernels.py:212-247): interior line (k, j) --
// Jacobi out of place (src -> dst, the i loop is parallel), GS in place on
// `src` (sequential along i, one thread).
__global__ void line_kernel(int kernel, const double* src, double* dst, int ni, int nj, int k, int j,
                            double a, double b) {
    const int64_t nip = ni + 2, plane = nip * (nj + 2);
    const int64_t base = (int64_t)(k + 1) * plane + (int64_t)(j + 1) * nip;
    if (kernel == SB_KERNEL_JACOBI) {
        for (int i = 1 + threadIdx.x; i <= ni; i += blockDim.x) {
            const double* c = src + base + i;
            double acc = __dadd_rn(c[-1], c[1]);
            acc = __dadd_rn(acc, c[-nip]);
            acc = __dadd_rn(acc, c[nip]);
            acc = __dadd_rn(acc, c[-plane]);
            acc = __dadd_rn(acc, c[plane]);
            dst[base + i] = __dadd_rn(__dmul_rn(a, c[0]), __dmul_rn(b, acc));
        }
        return;
    }
    if (threadIdx.x != 0) return;
    double* c = const_cast<double*>(src) + base;
    if (kernel == SB_KERNEL_GS_INTERLEAVED && ni >= 2) {
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

extern "C" int sb_line_update(int kernel, const double* src, double* dst, int64_t ni, int64_t nj,
                              int64_t nk, int64_t k, int64_t j, double a, double b, void* stream) {
    using namespace sb;
    clear_error();
    int rc = check_dims(ni, nj, nk);
    if (rc) return rc;
    if (kernel < SB_KERNEL_JACOBI || kernel > SB_KERNEL_GS_INTERLEAVED)
        return fail(SB_ERR_PLAN, "unknown kernel %d", kernel);
    if (k < 0 || k >= nk || j < 0 || j >= nj)
        return fail(SB_ERR_ARGUMENT, "line (k=%lld, j=%lld) outside interior of %lldx%lld planes",
                    (long long)k, (long long)j, (long long)nk, (long long)nj);
    if (!src || (kernel == SB_KERNEL_JACOBI && (!dst || dst == src)))
        return fail(SB_ERR_ARGUMENT, "Jacobi needs distinct src and dst");
    line_kernel<<<1, kernel == SB_KERNEL_JACOBI ? 256 : 32, 0, static_cast<cudaStream_t>(stream)>>>(
        kernel, src, dst, (int)ni, (int)nj, (int)k, (int)j, a, b);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? SB_OK : cuda_fail(e, "line kernel launch");
}
