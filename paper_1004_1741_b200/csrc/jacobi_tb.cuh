// jacobi_tb.cuh -- temporally blocked 3D 7-point Jacobi for sm_100a.
//
// One launch advances the field by T sweeps (T = 1 is the plain streaming
// sweep).  It is the B200 analogue of the reference's wavefront temporal
// blocking (reference sweeps/wavefront.py:160-312): there,
// t threads of a group each own one sweep and trail each other by two
// planes through a j-block held in the shared cache; here, the T "levels"
// of a CTA each own one sweep and trail each other by one plane through an
// xy tile held on chip.  Only level 1 reads HBM (TMA plane loads into a
// shared-memory ring) and only level T writes it, so HBM traffic is 16/T
// bytes per lattice-site update.
//
// Data placement (chosen from ncu: the first version was shared-memory
// bound, 82% of the LSU/smem pipe with 2-way bank conflicts):
//   * a warp spans the whole 64-cell tile width (lane = 2 cells, i-pairs),
//     so W/E neighbours are warp shuffles;
//   * a thread owns RJ consecutive rows, so N/S neighbours are registers,
//     except at warp-strip boundaries, which go through a small
//     double-buffered shared "exchange" row per warp and level;
//   * the z-queues (planes k-1, k, k+1 of the level below) live in
//     registers -- for level 1 optionally not: it can read the TMA ring
//     directly (JacobiCfg::L1S); levels trail by one plane, one
//     __syncthreads per plane;
//   * level T stages its output tile in shared memory and one thread writes
//     it with a TMA tensor store per plane (JacobiCfg::TS; the per-thread
//     alternative, coalesced 16-byte global stores, cost ~70 address
//     instructions per step that the compiler rematerialised under register
//     pressure).
// Overlapped (trapezoid) tiling: level L is valid on the tile grown by T-L
// cells; rows outside that region skip their arithmetic.
//
// Arithmetic (reference kernels.py:125-134):
//     v = a*c + b*(((((W+E)+S)+N)+D)+U)
// with explicit round-to-nearest intrinsics (no contraction; the library
// is also built with -fmad=false): bitwise equal to the reference for
// every T.  (A specialisation for a == 0 that drops a*c and patches the
// sign-of-zero / non-finite cases was measured slower: its integer checks
// cost more issue slots than the two DP operations they save.)  Halo (Dirichlet) cells are never computed: at every level they carry the
// input value.
//
// Work distribution: persistent CTAs claim (tile, k-range) items from a
// global atomic counter -- regular k-block-major items (CTAs running together
// hold neighbouring tiles of the same planes, so overlapping halo reads hit
// L2) or an explicit list built on the host (sched.cu: whole-k rounds with
// the border tiles first, then a balanced tail of k-pieces).  The TMA
// producer runs C::AHEAD planes ahead, across item boundaries.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>

#include "sb_ptx.cuh"

namespace sb {

// Halo planes sent straight from a slab launch into its neighbours' ghost
// planes (the fused z-slab exchange, sb_jacobi_slabs): output plane k in
// [k0[q], k1[q]) is also written, by the threads that computed it, to plane
// k + off[q] of buf[q] -- a buffer of the same plane shape on the
// neighbouring slab (peer memory over NVLink when that slab is on another
// GPU).  buf[q] == nullptr: no neighbour on that side.
struct JacPeers {
    double* buf[2];
    int k0[2], k1[2];
    int off[2];
};

struct JacobiParams {
    int ni, nj, nk;          // interior extents
    int kfirst, klast;       // output planes [kfirst, klast) (padded indices, within [1, nk])
    int tiles_i, tiles_j;    // output tiles per plane
    int kblk;                // planes per work item
    int kblocks;             // ceil((klast - kfirst) / kblk)
    int items;               // tiles_i * tiles_j * kblocks, or the length of `list`
    const int4* list;        // null: regular k-block-major items; else explicit items
                             // (tile, first plane, end plane, -) claimed in list order
    double a, b;
    int* counter;            // work counter (zeroed before launch)
    double* dst;             // output grid
    int64_t plane;           // (nj + 2) * (ni + 2) cells, < 2^31 (check_dims)
    JacPeers peers;          // fused halo exchange (zero: none)
};

template <int T_, int RJ_, int NW_, int S_, int MINB_, bool L1S_ = false, bool TS_ = false,
          bool UNI_ = false>
struct JacobiCfg {
    static constexpr int T = T_, RJ = RJ_, NW = NW_, S = S_, MINB = MINB_;
    // UNI: every step of an item in StepMode MASK (one inlined step loop)
    // instead of MASK / FAST-or-MASK / MASK segments: no FAST loop at all.
    // One loop instead of two leaves ptxas room for 5 rows per thread at
    // T = 4 without spilling.
    static constexpr bool UNI = UNI_;
    static constexpr bool LISTONLY = T_ >= 3 && T_ != 4;  // see decode_item
    // TS: level T writes its output tile into a shared staging buffer (double
    // buffered) and one thread stores it with a TMA tensor store per plane,
    // instead of per-thread 16-byte global stores
    static constexpr bool TS = TS_;
    // L1S: level 1 reads planes k-1, k, k+1 from the ring (three live slots,
    // prefetch distance S-2) instead of a register queue (prefetch S-1):
    // fewer registers (more warps / CTAs per SM), more shared-memory loads
    static constexpr bool L1S = L1S_;
    static constexpr int NQ = L1S ? (T > 1 ? T - 1 : 1) : T;  // register queues
    // TMA prefetch distance: the ring slots still being read limit it
    static constexpr int AHEAD = L1S ? S - 2 : S - 1;
    static_assert(AHEAD >= 1, "ring too small");
    static constexpr int H = (T + 1) / 2 * 2;          // input halo along i (even: TMA boxes
                                                       // must start 16-byte aligned)
    static constexpr int BW = 64;                      // cells per warp row (32 lanes x 2)
    static constexpr int TO = BW - 2 * H;              // output columns per tile (= i stride)
    static constexpr int ROWS = NW * RJ;               // rows computed per tile (level-1 region)
    static constexpr int TJ = ROWS - 2 * (T - 1);      // output rows per tile
    static_assert(TJ >= 1, "tile too short for this depth");
    static_assert(S_ >= (L1S_ ? 3 : 2), "ring too small");
    static constexpr int BH = ROWS + 2;                // input box rows (+1 neighbour row each side)
    static constexpr int BOX = BW * BH;
    static constexpr int BOXS = (BOX + 15) / 16 * 16;  // 128-B aligned TMA destinations
    static constexpr int NT = NW * 32;
    static constexpr int STORER = (NW - 1) * 32;       // thread issuing the output TMA stores
    static constexpr int XROW = 2 * BW;                // exchange doubles per warp: top + bottom row
    static constexpr int NX = (T > 1) ? (T - 1) : 0;   // levels with exchange rows (1..T-1)
    static constexpr int XSLOT = NW;                   // one slot per warp
    static constexpr int XB = 2;                       // exchange buffers (step parity)
    static constexpr int QSLOTS = 4;
    static constexpr size_t RING_OFF = 0;
    static constexpr size_t X_OFF = RING_OFF + size_t(S) * BOXS;
    static constexpr int STG = (TO * TJ + 15) / 16 * 16;  // staging doubles per buffer
    static constexpr size_t STG_OFF = X_OFF + size_t(NX) * XB * XSLOT * XROW;
    static constexpr size_t DBL_END = STG_OFF + (TS ? 2 * size_t(STG) : 0);
    // doubles, then queue[QSLOTS], mbarriers full[S], then the producer state
    static constexpr size_t SMEM_BYTES = DBL_END * 8 + 16 * QSLOTS + 8 * S + 32 + 64;
    static_assert(SMEM_BYTES <= 232448, "tile configuration exceeds 227 KB of shared memory");
    static constexpr uint32_t BOX_BYTES = uint32_t(BOX) * 8;
};

struct ItemInfo {
    int I0, J0;    // output tile origin (padded coordinates; I0 even)
    int kb, N;     // first output plane, number of plane steps (ke - kb + 2T); N == 0: stop
};

__device__ __forceinline__ double jac_cell(double a, double b, double c, double w, double e,
                                           double s, double n, double d, double u) {
    double acc = __dadd_rn(w, e);
    acc = __dadd_rn(acc, s);
    acc = __dadd_rn(acc, n);
    acc = __dadd_rn(acc, d);
    acc = __dadd_rn(acc, u);
    return __dadd_rn(__dmul_rn(a, c), __dmul_rn(b, acc));
}

template <class C>
__device__ __forceinline__ ItemInfo decode_item(const JacobiParams& p, int item) {
    ItemInfo it;
    if (item >= p.items) {
        it.I0 = it.J0 = it.kb = it.N = 0;
        return it;
    }
    int t, ke;
    // depths >= 3 always launch with an explicit list (sched.cu: item_list), so
    // their kernels need no arithmetic decode (two integer divisions inlined
    // at every item switch).  Dropping it changes ptxas' allocation: T=3 gains
    // 1.7% at 512^3, T=4 loses 0.6% (32 instead of 8 spill bytes), so the
    // T=4 kernel keeps both forms (profiles/r2/ab_list_only_decode.log).
    if (C::LISTONLY || p.list) {
        const int4 v = __ldg(p.list + item);
        t = v.x;
        it.kb = v.y;
        ke = v.z;
    } else {
        const int per_block = p.tiles_i * p.tiles_j;
        const int kbi = item / per_block;
        t = item - kbi * per_block;
        it.kb = p.kfirst + kbi * p.kblk;
        ke = min(it.kb + p.kblk, p.klast);
    }
    const int ti = t % p.tiles_i, tj = t / p.tiles_i;
    it.I0 = C::TO * ti;
    it.J0 = 1 + C::TJ * tj;
    it.N = ke - it.kb + 2 * C::T;
    return it;
}

__device__ __forceinline__ double2 lds2(const double* p) { return *reinterpret_cast<const double2*>(p); }
__device__ __forceinline__ void sts2(double* p, double x, double y) {
    *reinterpret_cast<double2*>(p) = make_double2(x, y);
}

// Fused halo exchange (JacobiParams::peers; kernels instantiated with PEER,
// used for a slab's edge-plane launches only): output plane k, staged in
// shared memory as the TO x TJ tile at (I0, J0), is copied by the whole CTA
// into the neighbour slab's ghost plane (peer memory over NVLink between
// GPUs).  The staging buffer is next overwritten two steps later, after
// another barrier.
template <class C>
__device__ __forceinline__ void peer_copy(const JacobiParams& p, const double* stg, int I0, int J0,
                                          int k) {
    constexpr int PAIRS = C::TO / 2;
#pragma unroll 1
    for (int q = 0; q < 2; ++q) {
        if (!p.peers.buf[q] || k < p.peers.k0[q] || k >= p.peers.k1[q]) continue;
        double* plane = p.peers.buf[q] + (int64_t)(k + p.peers.off[q]) * p.plane;
        for (int x = threadIdx.x; x < C::TJ * PAIRS; x += C::NT) {
            const int row = x / PAIRS, i2 = 2 * (x - row * PAIRS);
            const int gj = J0 + row, gi = I0 + i2;
            if (gj <= p.nj && gi <= p.ni)  // inside the grid (gi + 1 <= ni + 1)
                *reinterpret_cast<double2*>(plane + (int64_t)gj * (p.ni + 2) + gi) =
                    lds2(stg + row * C::TO + i2);
        }
    }
}

// Per-thread state of one level's input: three plane slots rotating with
// the step phase (D, C, U = slots PH, PH+1, PH+2 mod 3), RJ rows x 2 cells.
template <class C>
struct LevelQ {
    double q[3][C::RJ][2];
};

// The final operation of a cell.  Reference: RN(RN(a*c) + RN(b*acc)).  When
// a == +-0 the product a*c is exact (a signed zero, or NaN for non-finite
// c), so RN(a*c + RN(b*acc)) -- one fused multiply-add -- is the same value
// bit for bit, including signed zeros and NaNs; it saves one DP operation.
template <bool AZ>
__device__ __forceinline__ double jac_final(double a, double b, double c, double acc) {
    if (AZ) return __fma_rn(a, c, __dmul_rn(b, acc));
    return __dadd_rn(__dmul_rn(a, c), __dmul_rn(b, acc));
}

struct JState {      // per-thread loop state shared by the step functions
    uint32_t g;      // global plane-step counter (exchange parity, rotation)
    int slot;        // ring slot of step g (= g mod S) and its mbarrier phase parity,
    uint32_t phase;  // kept incrementally when S is not a power of two
    int n, cq;       // step within the item, consumer queue slot
    ItemInfo it;     // current item
    uint32_t ooff;   // this thread's output cell (row 0) within a plane
    uint32_t omask;  // bit r: row r of this thread is an output row of the current item
    uint32_t keep0, keep1;  // bit r: cell 0 / 1 of row r is a Dirichlet cell (MASK steps)
    uint32_t smask;  // TS: bit r: row r of this thread lies in the staged output tile
    int soff;        // TS: staging offset of this thread's row 0
};

// The TMA producer's state.  Only thread 0 produces, so it lives in shared
// memory instead of occupying registers in every thread: two 16-byte records
// (counters, current item), each read with one load per step.
struct alignas(16) Prod {
    uint32_t ld_issued;  // plane loads issued
    int pq, pn;          // queue slot / plane step of the producer's item
    int pad;
    ItemInfo pitem;      // producer's item
};

// Per-item output addressing of a thread (hoisted out of the plane steps).
template <class C>
__device__ __forceinline__ void item_output(const JacobiParams& p, JState& s) {
    const int tid = threadIdx.x;
    const int lane = tid & 31, w = tid >> 5;
    const int di = 2 * lane - C::H;
    const int dj = -(C::T - 1) + w * C::RJ;
    const int gi = s.it.I0 + di, gj = s.it.J0 + dj;
    if (!C::TS) {
        uint32_t m = 0;
        if (di >= 0 && di < C::TO && gi + 1 <= p.ni + 1) {
#pragma unroll
            for (int r = 0; r < C::RJ; ++r)
                if (dj + r >= 0 && dj + r < C::TJ && gj + r <= p.nj) m |= 1u << r;
        }
        s.omask = m;
        s.ooff = uint32_t(gj * (p.ni + 2) + gi);
    }
    uint32_t rows_out = 0;
#pragma unroll
    for (int r = 0; r < C::RJ; ++r)
        if (gj + r < 1 || gj + r > p.nj) rows_out |= 1u << r;
    const uint32_t all = (1u << C::RJ) - 1;
    s.keep0 = rows_out | ((gi >= 1 && gi <= p.ni) ? 0u : all);
    s.keep1 = rows_out | ((gi + 1 >= 1 && gi + 1 <= p.ni) ? 0u : all);
}

// The producer's next work item.
template <class C>
__device__ __forceinline__ void next_item(const JacobiParams& p, ItemInfo* queue, Prod& pr) {
    pr.pitem = decode_item<C>(p, atomicAdd(p.counter, 1));
    queue[pr.pq] = pr.pitem;
}

// Prod sits between the item queue and the mbarriers (16-byte aligned).
template <class C>
__device__ __forceinline__ Prod* prod_state(ItemInfo* queue) {
    return reinterpret_cast<Prod*>(queue + C::QSLOTS);
}

// One plane load of the producer's item into the ring slot of load number
// ld_issued.  The whole state is read up front (two independent 16-byte
// shared loads) and kept in registers across the mbarrier / TMA
// instructions: thread 0 carries this after every step barrier, and every
// dependent shared-memory round trip here delays warp 0 -- and, through the
// next barrier, the CTA.
template <class C>
__device__ __forceinline__ void produce(const CUtensorMap* src_map, const JacobiParams& p,
                                        double* ring, uint64_t* full, ItemInfo* queue) {
    constexpr int S = C::S;
    Prod& pr = *prod_state<C>(queue);
    const int4 cnt = *reinterpret_cast<const int4*>(&pr);         // ld_issued, pq, pn, -
    const int4 itm = *reinterpret_cast<const int4*>(&pr.pitem);  // I0, J0, kb, N
    if (itm.w <= 0) return;
    const uint32_t ld = uint32_t(cnt.x);
    const int slot = int(ld % S);
    uint64_t* bar = &full[slot];
    mbar_arrive_expect_tx(bar, C::BOX_BYTES);
    tma_load_3d(ring + size_t(slot) * C::BOXS, src_map, itm.x - C::H, itm.y - C::T,
                itm.z - C::T + cnt.z, bar);
    if (cnt.z + 1 == itm.w) {
        pr.ld_issued = ld + 1;
        pr.pn = 0;
        pr.pq = (cnt.y + 1) % C::QSLOTS;
        next_item<C>(p, queue, pr);
    } else {
        pr.ld_issued = ld + 1;
        pr.pn = cnt.z + 1;
    }
}

// Step modes.  FAST: every cell the tile computes at this step is interior
// (no masks).  MASK: any step -- the same two-phase arithmetic everywhere,
// then Dirichlet cells (the item's i/j masks, plus every cell of a level
// whose plane lies outside [1, nk]) keep their value.  Cells outside a
// level's trapezoid then hold values that no output depends on (level L+1
// reads level L only inside its own, smaller, trapezoid grown by one cell).
// MASK replaced round 1's one-pass SLOW (full predication; k-boundary steps
// and tiny grids) and SEL (border tiles): +3% at 512^3 where every whole-k
// item has 2(2T+1) k-boundary steps (profiles/r2/ab_mask_modes.log).
enum StepMode { FAST = 1, MASK = 3 };

// Phase 1 of a level: the partial sums P = ((((W+E)+S)+N)+D) of the RJ rows
// x 2 cells.  cen: the centre plane with the south (row 0) and north (row
// RJ+1) neighbour rows; dn: the plane below.  P may alias dn.
template <class C>
__device__ __forceinline__ void level_partial(const double (&cen)[C::RJ + 2][2],
                                              const double (&dn)[C::RJ][2],
                                              double (&P)[C::RJ][2]) {
#pragma unroll
    for (int r = 0; r < C::RJ; ++r) {
        const double c0 = cen[r + 1][0], c1 = cen[r + 1][1];
        const double wv = __shfl_up_sync(0xffffffffu, c1, 1);    // cell i-1 (lane-1)
        const double ev = __shfl_down_sync(0xffffffffu, c0, 1);  // cell i+2 (lane+1)
        double acc0 = __dadd_rn(wv, c1), acc1 = __dadd_rn(c0, ev);
        acc0 = __dadd_rn(acc0, cen[r][0]);
        acc1 = __dadd_rn(acc1, cen[r][1]);
        acc0 = __dadd_rn(acc0, cen[r + 2][0]);
        acc1 = __dadd_rn(acc1, cen[r + 2][1]);
        P[r][0] = __dadd_rn(acc0, dn[r][0]);
        P[r][1] = __dadd_rn(acc1, dn[r][1]);
    }
}

// Phase 2 of a level: v = a*c + b*(P + U) (the reference association, see
// jac_final), then the step mode's Dirichlet handling (k: the level's plane).
template <class C, int MODE, bool AZ>
__device__ __forceinline__ void level_finish(const double (&cc)[C::RJ][2],
                                             const double (&P)[C::RJ][2],
                                             const double (&up)[C::RJ][2], double (&nv)[C::RJ][2],
                                             double a, double b, int k, const JacobiParams& p,
                                             const JState& s) {
    constexpr int RJ = C::RJ;
#pragma unroll
    for (int r = 0; r < RJ; ++r) {
        const double c0 = cc[r][0], c1 = cc[r][1];
        const double o0 = jac_final<AZ>(a, b, c0, __dadd_rn(P[r][0], up[r][0]));
        const double o1 = jac_final<AZ>(a, b, c1, __dadd_rn(P[r][1], up[r][1]));
        if (MODE == FAST) {
            nv[r][0] = o0;
            nv[r][1] = o1;
        } else {
            const uint32_t kall = (k < 1 || k > p.nk) ? 0xffffffffu : 0u;  // CTA-uniform
            nv[r][0] = ((s.keep0 | kall) & (1u << r)) ? c0 : o0;
            nv[r][1] = ((s.keep1 | kall) & (1u << r)) ? c1 : o1;
        }
    }
}

// One plane step of the current item in StepMode MODE.  PH = g mod 3
// selects the register rotation statically.  With C::L1S level 1 reads its
// three input planes straight from the TMA ring (slots g-2, g-1, g);
// otherwise from register queue Q[0], fed from ring slot g.
//
// Steps run in two phases.  Phase 1 forms every level's partial sum P
// from data of the previous step only (centre and lower planes in registers, neighbour rows in
// the exchange buffers / ring) -- T x RJ x 2 independent chains, so the
// shuffles and adds of all levels overlap.  P overwrites the lower plane,
// which nothing else needs.  Phase 2 is the short dependent chain through the
// levels: level L's new plane is level L+1's U.
template <class C, int MODE, bool AZ, int PH, bool PEER>
__device__ __forceinline__ bool jacobi_step(const CUtensorMap* src_map, const CUtensorMap* dst_map,
                                            const JacobiParams& p,
                                            double* ring, double* xb, uint64_t* full,
                                            ItemInfo* queue, LevelQ<C> (&Q)[C::NQ],
                                            JState& s) {
    constexpr int T = C::T, RJ = C::RJ, NW = C::NW, S = C::S, BW = C::BW;
    constexpr int D = PH % 3, CC = (PH + 1) % 3, U = (PH + 2) % 3;
    const int tid = threadIdx.x;
    const int lane = tid & 31, w = tid >> 5;
    const int col = 2 * lane;
    const int brow = 1 + w * RJ;
    const int di = col - C::H;
    const int dj = -(T - 1) + w * RJ;
    const ItemInfo& it = s.it;
    // exchange buffers: written this step / written by the previous step
    const int xwb = int(s.g & 1), xrb = int((s.g + 1) & 1);

    // ring slot of this step (power-of-two S: mask and shift of g, else the
    // incrementally kept slot -- a division by S every step costs issue slots)
    constexpr bool POW2 = (S & (S - 1)) == 0;
    const int slot = POW2 ? int(s.g & (S - 1)) : s.slot;
    const uint32_t phase = POW2 ? (s.g / S) & 1u : s.phase;
    const double* cur = ring + size_t(slot) * C::BOXS;
    const double* prv = ring + size_t(slot >= 1 ? slot - 1 : slot + S - 1) * C::BOXS;
    const double* pp = ring + size_t(slot >= 2 ? slot - 2 : slot + S - 2) * C::BOXS;
    const int pplane = it.kb - T + s.n;
    const double a = p.a, b = p.b;

    // emits level L's new plane: exchange rows + queue (L < T) or output
    auto emit = [&](int L, const double (&nv)[RJ][2]) {
        const int k = pplane - L;
        if (L < T) {
            double* xl = xb + size_t((L - 1) * C::XB + xwb) * C::XSLOT * C::XROW;
            double* xw = xl + w * C::XROW;
            sts2(xw + col, nv[0][0], nv[0][1]);
            sts2(xw + BW + col, nv[RJ - 1][0], nv[RJ - 1][1]);
#pragma unroll
            for (int r = 0; r < RJ; ++r) {
                Q[C::L1S ? L - 1 : L].q[U][r][0] = nv[r][0];
                Q[C::L1S ? L - 1 : L].q[U][r][1] = nv[r][1];
            }
        } else if (C::TS) {
            if (s.n >= 2 * T && s.smask) {
                double* stg = ring + C::STG_OFF + (s.g & 1) * C::STG;
#pragma unroll
                for (int r = 0; r < RJ; ++r)
                    if (s.smask & (1u << r)) sts2(stg + s.soff + r * C::TO, nv[r][0], nv[r][1]);
            }
        } else if (s.n >= 2 * T && s.omask) {
            double* plane = p.dst + (int64_t)k * p.plane;  // CTA-uniform
            uint32_t o = s.ooff;
#pragma unroll
            for (int r = 0; r < RJ; ++r) {
                if (s.omask & (1u << r))
                    *reinterpret_cast<double2*>(plane + o) = make_double2(nv[r][0], nv[r][1]);
                o += uint32_t(p.ni + 2);
            }
        }
    };
    // the centre plane's neighbour rows of level L
    auto nbr_rows = [&](int L, double (&cen)[RJ + 2][2]) {
        double2 s2, n2;
        if (L == 1) {  // from the ring
            s2 = lds2(prv + (brow - 1) * BW + col);
            n2 = lds2(prv + (brow + RJ) * BW + col);
        } else {
            // south: bottom row of warp w-1, north: top row of warp w+1
            // (clamped at the tile edge: those rows lie outside the trapezoid
            // and their values are never used)
            const double* xr = xb + size_t((L - 2) * C::XB + xrb) * C::XSLOT * C::XROW;
            s2 = lds2(xr + max(w - 1, 0) * C::XROW + BW + col);
            n2 = lds2(xr + min(w + 1, NW - 1) * C::XROW + col);
        }
        cen[0][0] = s2.x;
        cen[0][1] = s2.y;
        cen[RJ + 1][0] = n2.x;
        cen[RJ + 1][1] = n2.y;
    };

    {
        // ---- phase 1: partial sums of every level (previous-step data) ----
        double P1[RJ][2], C1[RJ][2];  // L1S: level 1's P and centre plane (else unused)
#pragma unroll
        for (int L = 1; L <= T; ++L) {
            double cen[RJ + 2][2];
            nbr_rows(L, cen);
            if (C::L1S && L == 1) {
                double dn[RJ][2];
#pragma unroll
                for (int r = 0; r < RJ; ++r) {
                    const double2 x = lds2(prv + (brow + r) * BW + col);
                    const double2 y = lds2(pp + (brow + r) * BW + col);
                    cen[r + 1][0] = C1[r][0] = x.x;
                    cen[r + 1][1] = C1[r][1] = x.y;
                    dn[r][0] = y.x;
                    dn[r][1] = y.y;
                }
                level_partial<C>(cen, dn, P1);
            } else {
                LevelQ<C>& In = Q[C::L1S ? L - 2 : L - 1];
#pragma unroll
                for (int r = 0; r < RJ; ++r) {
                    cen[r + 1][0] = In.q[CC][r][0];
                    cen[r + 1][1] = In.q[CC][r][1];
                }
                level_partial<C>(cen, In.q[D], In.q[D]);
            }
        }
        // ---- phase 2: the level chain ----
        mbar_wait(&full[slot], phase);
        double U1[RJ][2];
#pragma unroll
        for (int r = 0; r < RJ; ++r) {
            const double2 x = lds2(cur + (brow + r) * BW + col);
            U1[r][0] = x.x;
            U1[r][1] = x.y;
        }
#pragma unroll
        for (int L = 1; L <= T; ++L) {
            double nv[RJ][2];
            if (C::L1S && L == 1) {
                level_finish<C, MODE, AZ>(C1, P1, U1, nv, a, b, pplane - L, p, s);
            } else {
                LevelQ<C>& In = Q[C::L1S ? L - 2 : L - 1];
                if (L == 1) {
#pragma unroll
                    for (int r = 0; r < RJ; ++r) {
                        In.q[U][r][0] = U1[r][0];
                        In.q[U][r][1] = U1[r][1];
                    }
                }
                level_finish<C, MODE, AZ>(In.q[CC], In.q[D], In.q[U], nv, a, b, pplane - L, p, s);
            }
            emit(L, nv);
        }
    }
    const bool out_step = s.n >= 2 * T;
    if (C::TS && out_step) {
        fence_proxy_async_smem();  // staged rows -> visible to the TMA store
        // the store issued last step has read the other staging buffer, which
        // the next step overwrites
        if (tid == C::STORER) bulk_wait_read<0>();
    }
    __syncthreads();
    // fused halo exchange: an edge output plane, staged in shared memory, is
    // also copied by the whole CTA into the neighbour slab's ghost plane
    // (CTA-uniform; only the `depth` edge planes of a slab launch).  The
    // staging buffer is next overwritten two steps later, after another
    // barrier.
    if constexpr (PEER) {
        if (out_step) peer_copy<C>(p, ring + C::STG_OFF + (s.g & 1) * C::STG, it.I0, it.J0,
                                   it.kb - 2 * T + s.n);
    }
    // the per-step TMA duties after the barrier delay the warps that carry
    // them into the next step (and so, through the next barrier, everyone):
    // the output store goes to the last warp, the loads to warp 0
    if (C::TS && out_step && tid == C::STORER) {
        tma_store_3d(dst_map, ring + C::STG_OFF + (s.g & 1) * C::STG, it.I0, it.J0,
                     it.kb - 2 * T + s.n);
        bulk_commit();
    }
    // the oldest ring slot (g-2 with L1S, else g-1) is free now: refill it
    if (tid == 0) produce<C>(src_map, p, ring, full, queue);
    ++s.g;
    if (!POW2 && ++s.slot == S) {
        s.slot = 0;
        s.phase ^= 1u;
    }
    return ++s.n == it.N;
}

// `count` plane steps of the current item (all in one StepMode),
// entering the 3-phase register rotation at g mod 3.
template <class C, int MODE, bool AZ, bool PEER>
__device__ __forceinline__ void jacobi_steps(const CUtensorMap* src_map, const CUtensorMap* dst_map,
                                             const JacobiParams& p,
                                             double* ring, double* xb, uint64_t* full,
                                             ItemInfo* queue, LevelQ<C> (&Q)[C::NQ],
                                             JState& s, int count) {
    if (count <= 0) return;
    const int ph = s.g % 3;
    if (ph == 1) {
        jacobi_step<C, MODE, AZ, 1, PEER>(src_map, dst_map, p, ring, xb, full, queue, Q, s);
        if (--count == 0) return;
        jacobi_step<C, MODE, AZ, 2, PEER>(src_map, dst_map, p, ring, xb, full, queue, Q, s);
        if (--count == 0) return;
    } else if (ph == 2) {
        jacobi_step<C, MODE, AZ, 2, PEER>(src_map, dst_map, p, ring, xb, full, queue, Q, s);
        if (--count == 0) return;
    }
    while (true) {
        jacobi_step<C, MODE, AZ, 0, PEER>(src_map, dst_map, p, ring, xb, full, queue, Q, s);
        if (--count == 0) return;
        jacobi_step<C, MODE, AZ, 1, PEER>(src_map, dst_map, p, ring, xb, full, queue, Q, s);
        if (--count == 0) return;
        jacobi_step<C, MODE, AZ, 2, PEER>(src_map, dst_map, p, ring, xb, full, queue, Q, s);
        if (--count == 0) return;
    }
}

// The same from a step with g mod 3 == 0: no prologue, so each step
// variant is inlined once per call site (the kernel's instruction-cache
// footprint matters: profiles/r2/ab_phase_aligned.log).
template <class C, int MODE, bool AZ, bool PEER>
__device__ __forceinline__ void jacobi_steps0(const CUtensorMap* src_map, const CUtensorMap* dst_map,
                                              const JacobiParams& p,
                                              double* ring, double* xb, uint64_t* full,
                                              ItemInfo* queue, LevelQ<C> (&Q)[C::NQ],
                                              JState& s, int count) {
    while (count > 0) {
        jacobi_step<C, MODE, AZ, 0, PEER>(src_map, dst_map, p, ring, xb, full, queue, Q, s);
        if (--count == 0) return;
        jacobi_step<C, MODE, AZ, 1, PEER>(src_map, dst_map, p, ring, xb, full, queue, Q, s);
        if (--count == 0) return;
        jacobi_step<C, MODE, AZ, 2, PEER>(src_map, dst_map, p, ring, xb, full, queue, Q, s);
        --count;
    }
}

template <class C, bool AZ, bool PEER = false>
__global__ void __launch_bounds__(C::NT, C::MINB)
jacobi_tb_kernel(const __grid_constant__ CUtensorMap src_map,
                 const __grid_constant__ CUtensorMap dst_map, const JacobiParams p) {
    constexpr int T = C::T, S = C::S;
    extern __shared__ __align__(128) double smem[];
    double* ring = smem + C::RING_OFF;
    double* xb = smem + C::X_OFF;
    // queue[QSLOTS] (16-byte entries, 128-byte aligned), the producer state, full[S]
    ItemInfo* queue = reinterpret_cast<ItemInfo*>(smem + C::DBL_END);
    uint64_t* full = reinterpret_cast<uint64_t*>(prod_state<C>(queue) + 1);
    const int tid = threadIdx.x;

    JState s;
    if (tid == 0) {
        tma_prefetch_desc(&src_map);
        if (C::TS) tma_prefetch_desc(&dst_map);
        for (int i = 0; i < S; ++i) mbar_init(&full[i], 1);
        fence_mbar_init();
    }
    if (tid == 0) {
        Prod& pr = *prod_state<C>(queue);
        pr.ld_issued = 0;
        pr.pq = pr.pn = 0;
        next_item<C>(p, queue, pr);
        while (pr.ld_issued < C::AHEAD && pr.pitem.N > 0) produce<C>(&src_map, p, ring, full, queue);
    }
    __syncthreads();

    LevelQ<C> Q[C::NQ];
#pragma unroll
    for (int L = 0; L < C::NQ; ++L)
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int r = 0; r < C::RJ; ++r) Q[L].q[i][r][0] = Q[L].q[i][r][1] = 0.0;

    s.g = 0;
    s.slot = 0;
    s.phase = 0;
    s.n = 0;
    s.cq = 0;
    s.it = queue[0];
    if (C::TS) {  // this thread's cells in the staged TO x TJ output tile (item-invariant)
        const int lane = tid & 31, w = tid >> 5;
        const int di = 2 * lane - C::H, dj = -(T - 1) + w * C::RJ;
        uint32_t m = 0;
        if (di >= 0 && di < C::TO) {
#pragma unroll
            for (int r = 0; r < C::RJ; ++r)
                if (dj + r >= 0 && dj + r < C::TJ) m |= 1u << r;
        }
        s.smask = m;
        s.soff = dj * C::TO + di;
    }
    while (s.it.N > 0) {
        item_output<C>(p, s);
        // Steps [n_lo, n_hi) compute interior planes only (step n computes
        // planes kb-T+n-L for L = 1..T; only the first/last steps of items
        // touching the k boundary are outside).  They run FAST when the
        // tile's rows and columns lie inside [1,nj] x [1,ni]; every other
        // step runs MASK.
        const int jlo = s.it.J0 - (T - 1);  // the tile's first computed row
        const bool ij_in = (s.it.I0 - C::H >= 1) && (s.it.I0 - C::H + C::BW - 1 <= p.ni) &&
                           (jlo >= 1) && (jlo + C::ROWS - 1 <= p.nj);
        const int n_lo = min(s.it.N, max(0, 2 * T + 1 - s.it.kb));
        const int n_hi = max(n_lo, min(s.it.N, p.nk + 2 + T - s.it.kb));
        if constexpr (C::UNI) {
            jacobi_steps<C, MASK, AZ, PEER>(&src_map, &dst_map, p, ring, xb, full, queue, Q, s, s.it.N);
        } else {
            // MASK (exact on any step) up to the first step with g mod 3 == 0
            // at or after n_lo, then FAST in whole rotations, then MASK: the
            // FAST and tail loops start at phase 0 and need no prologue
            int n1 = s.it.N;
            if (ij_in) n1 = min(s.it.N, n_lo + int((3u - (s.g + n_lo) % 3u) % 3u));
            jacobi_steps<C, MASK, AZ, PEER>(&src_map, &dst_map, p, ring, xb, full, queue, Q, s, n1);
            const int nf = max(0, n_hi - n1) / 3 * 3;
            jacobi_steps0<C, FAST, AZ, PEER>(&src_map, &dst_map, p, ring, xb, full, queue, Q, s, nf);
            jacobi_steps0<C, MASK, AZ, PEER>(&src_map, &dst_map, p, ring, xb, full, queue, Q, s,
                                             s.it.N - n1 - nf);
        }
        s.n = 0;
        __syncthreads();  // queue[] entry written by thread 0 at least one barrier ago
        s.cq = (s.cq + 1) % C::QSLOTS;
        s.it = queue[s.cq];
    }
    if (C::TS && tid == C::STORER) bulk_wait<0>();  // every output plane written before exit
}

}  // namespace sb
