// jacobi_tb.cuh -- temporally blocked 3D 7-point Jacobi for sm_100a.
//
// One launch advances the field by T sweeps (T = 1 is the plain streaming
// sweep).  It is the B200 analogue of the reference's wavefront temporal
// blocking (reference sweeps/wavefront.py:160-312): there,
// t threads of a group each own one sweep and trail each other by two
// planes through a j-block held in the shared cache; here, the T "levels"
// of a CTA each own one sweep and trail each other by one plane through an
// xy tile held in shared memory.  Only the first level reads HBM (TMA plane
// loads) and only the last writes it (TMA plane stores), so HBM traffic is
// 16/T bytes per lattice-site update.
//
// Tiling: an output tile is (TI+2) x TJ cells of an xy plane (tiles start
// every TI columns at even i; see JacobiCfg::TO), over a range of z-planes
// [kb, ke).  The input box of a plane is (TI+2+2H) x (TJ+2T) with
// H = T rounded up to even (overlapped/trapezoid halo: level L is valid on
// the box shrunk by L cells, so level T is valid on the output tile).  Each
// thread owns a 2(i) x RJ(j) block of cells at every level, keeps each
// level's z-queue (planes k-1, k, k+1 of the level below) in registers and
// exchanges in-plane neighbours through one double-buffered smem plane per
// level.  One __syncthreads per plane step.
//
// Arithmetic (reference kernels.py:125-134):
//     v = a*c + b*(((((W+E)+S)+N)+D)+U)
// with explicit round-to-nearest intrinsics (no FMA contraction; the
// library is also built with -fmad=false), so results are bitwise equal to
// the reference for every T.  Halo (Dirichlet) cells are never computed:
// at every level they carry the input value, and the output keeps them.
//
// Work distribution: persistent CTAs grab (tile, k-block) items from a
// global atomic counter, in k-block-major order so that CTAs working at the
// same time hold neighbouring tiles of the same planes (their overlapping
// halo reads hit L2).  The TMA producer runs S-1 plane steps ahead of the
// compute, across item boundaries, so the pipeline never drains between
// items.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>

#include "sb_ptx.cuh"

namespace sb {

struct JacobiParams {
    int ni, nj, nk;          // interior extents
    int kfirst, klast;       // output planes [kfirst, klast) (padded indices, within [1, nk])
    int tiles_i, tiles_j;    // output tiles per plane
    int kblk;                // planes per work item
    int kblocks;             // ceil(nk / kblk)
    int items;               // tiles_i * tiles_j * kblocks
    double a, b;
    int* counter;            // work counter (zeroed before launch)
};

template <int T_, int TI_, int TJ_, int RJ_, int S_, int MINB_>
struct JacobiCfg {
    static constexpr int T = T_, TI = TI_, TJ = TJ_, RJ = RJ_, S = S_, MINB = MINB_;
    // Along i every TMA box must start on an even index (16-byte aligned
    // fp64 rows), so tiles start at even padded i (stride TI) and write
    // TO = TI + 2 columns; neighbouring tiles overlap by two columns and
    // write bitwise-identical values there.
    static constexpr int TO = TI + 2;                  // output columns per tile
    static constexpr int H = (T + 1) / 2 * 2;          // input halo along i (even)
    static constexpr int HP = (T - 1 + 1) / 2 * 2;     // computed halo along i at level 1 (even)
    static constexpr int BW = TO + 2 * H;              // input box width
    static constexpr int BH = TJ + 2 * T;              // input box rows
    static constexpr int PLANE = BW * BH;              // doubles per plane buffer
    static constexpr int PSTRIDE = (PLANE + 15) / 16 * 16;  // 128-B aligned (TMA destination)
    static constexpr int TC = TO / 2 + HP;             // thread columns (cell pairs)
    static constexpr int ROWS1 = TJ + 2 * (T - 1);     // rows computed at level 1
    static_assert(ROWS1 % RJ == 0, "rows per thread must divide the level-1 row count");
    static constexpr int TR = ROWS1 / RJ;              // thread rows
    static constexpr int NT = TC * TR;                 // threads per CTA
    static constexpr int OUT = TO * TJ;                // doubles per output tile
    static constexpr int NLVL = (T > 1) ? (T - 1) : 0; // smem level planes (levels 1..T-1)
    static constexpr int QSLOTS = 4;                   // item queue depth
    // smem layout (in doubles): ring[S] | lvl[NLVL][2] | out[2] ; then barriers + item queue
    static constexpr size_t RING_OFF = 16;             // 128-B guard before the first buffer
    static constexpr size_t LVL_OFF = RING_OFF + size_t(S) * PSTRIDE;
    static constexpr size_t OUT_OFF = LVL_OFF + size_t(NLVL) * 2 * PSTRIDE;
    static constexpr size_t DBL_END = OUT_OFF + 2 * size_t((OUT + 15) / 16 * 16);
    static constexpr size_t SMEM_BYTES = DBL_END * 8 + 8 * S + 16 * QSLOTS + 64;
    static constexpr uint32_t BOX_BYTES = uint32_t(BW) * BH * 8;
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
    const int per_block = p.tiles_i * p.tiles_j;
    const int kbi = item / per_block;
    const int t = item - kbi * per_block;
    const int ti = t % p.tiles_i, tj = t / p.tiles_i;
    it.I0 = C::TI * ti;
    it.J0 = 1 + C::TJ * tj;
    it.kb = p.kfirst + kbi * p.kblk;
    const int ke = min(it.kb + p.kblk, p.klast);
    it.N = ke - it.kb + 2 * C::T;
    return it;
}

template <class C>
__global__ void __launch_bounds__(C::NT, C::MINB)
jacobi_tb_kernel(const __grid_constant__ CUtensorMap src_map,
                 const __grid_constant__ CUtensorMap dst_map, const JacobiParams p) {
    constexpr int T = C::T, TI = C::TI, TJ = C::TJ, RJ = C::RJ, S = C::S;
    constexpr int BW = C::BW, PSTRIDE = C::PSTRIDE;
    extern __shared__ __align__(128) double smem[];
    double* ring = smem + C::RING_OFF;
    double* lvl = smem + C::LVL_OFF;
    double* outb = smem + C::OUT_OFF;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::DBL_END);
    ItemInfo* queue = reinterpret_cast<ItemInfo*>(full + S);

    const int tid = threadIdx.x;
    const int tx = tid % C::TC, ty = tid / C::TC;
    // smem column of this thread's first cell, smem row of its first row
    const int c0 = C::H - C::HP + 2 * tx;
    const int r0 = 1 + RJ * ty;
    // offsets of this thread's cells relative to the tile origin
    const int di = -C::HP + 2 * tx;        // i - I0 of the first cell
    const int dj = -(T - 1) + RJ * ty;     // j - J0 of the first row

    // ---- producer state (thread 0 only) ------------------------------------
    uint32_t ld_issued = 0;    // loads issued so far (slot = count % S)
    int pq = 0;                // producer queue slot of its current item
    ItemInfo pitem;
    int pn = 0;                // producer's plane step within its item

    if (tid == 0) {
        tma_prefetch_desc(&src_map);
        tma_prefetch_desc(&dst_map);
        for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
        pitem = decode_item<C>(p, atomicAdd(p.counter, 1));
        queue[0] = pitem;
        // prologue: fill S-1 ring slots
        while (ld_issued < S - 1 && pitem.N > 0) {
            uint64_t* bar = &full[ld_issued % S];
            mbar_arrive_expect_tx(bar, C::BOX_BYTES);
            tma_load_3d(ring + size_t(ld_issued % S) * PSTRIDE, &src_map, pitem.I0 - C::H,
                        pitem.J0 - T, pitem.kb - T + pn, bar);
            ++ld_issued;
            if (++pn == pitem.N) {
                pn = 0;
                pq = (pq + 1) % C::QSLOTS;
                pitem = decode_item<C>(p, atomicAdd(p.counter, 1));
                queue[pq] = pitem;
            }
        }
    }
    __syncthreads();

    // ---- consumer state -----------------------------------------------------
    // z-queues per level: level L values (L = 0..T-1) at planes k-1 (D) and k (C)
    double qD[T][RJ][2], qC[T][RJ][2];
#pragma unroll
    for (int L = 0; L < T; ++L)
#pragma unroll
        for (int r = 0; r < RJ; ++r) qD[L][r][0] = qD[L][r][1] = qC[L][r][0] = qC[L][r][1] = 0.0;

    uint32_t consumed = 0;  // global plane step counter
    int cq = 0;             // consumer queue slot
    ItemInfo it = queue[0];
    int n = 0;              // plane step within the current item

    while (it.N > 0) {
        const int slot = consumed % S;
        const int pslot = (consumed + S - 1) % S;
        mbar_wait(&full[slot], (consumed / S) & 1);
        const double* cur = ring + size_t(slot) * PSTRIDE;     // input plane p_n
        const double* prv = ring + size_t(pslot) * PSTRIDE;    // input plane p_n - 1
        const int pplane = it.kb - T + n;                      // newest input plane index

        // in-plane interior masks for this thread's cells
        const int gi = it.I0 + di, gj = it.J0 + dj;
        bool in_i[2], in_j[RJ];
        in_i[0] = (gi >= 1) && (gi <= p.ni);
        in_i[1] = (gi + 1 >= 1) && (gi + 1 <= p.ni);
#pragma unroll
        for (int r = 0; r < RJ; ++r) in_j[r] = (gj + r >= 1) && (gj + r <= p.nj);

        // level-0 values (own cells of the newest plane)
        double v[RJ][2];
#pragma unroll
        for (int r = 0; r < RJ; ++r) {
            const double2 x = *reinterpret_cast<const double2*>(cur + (r0 + r) * BW + c0);
            v[r][0] = x.x;
            v[r][1] = x.y;
        }

#pragma unroll
        for (int L = 1; L <= T; ++L) {
            const int kL = pplane - L;  // plane computed by level L at this step
            const bool kin = (kL >= 1) && (kL <= p.nk);
            // region of level L actually needed downstream: tile +- (T-L)
            const int need = T - L;
            const bool act = (di + 1 >= -need) && (di < C::TO + need) && (dj + RJ - 1 >= -need) &&
                             (dj < TJ + need);
            const double* src = (L == 1) ? prv : (lvl + size_t((L - 2) * 2 + ((consumed + 1) & 1)) * PSTRIDE);
            double nv[RJ][2];
            if (act) {
#pragma unroll
                for (int r = 0; r < RJ; ++r) {
                    const double* row = src + (r0 + r) * BW + c0;
                    const double w = row[-1];
                    const double e = row[2];
                    const double2 sv = *reinterpret_cast<const double2*>(row - BW);
                    const double2 nn = *reinterpret_cast<const double2*>(row + BW);
                    const double cc0 = qC[L - 1][r][0], cc1 = qC[L - 1][r][1];
                    // cell 0: W = w, E = cc1 (own neighbour), cell 1: W = cc0, E = e
                    double o0 = jac_cell(p.a, p.b, cc0, w, cc1, sv.x, nn.x, qD[L - 1][r][0], v[r][0]);
                    double o1 = jac_cell(p.a, p.b, cc1, cc0, e, sv.y, nn.y, qD[L - 1][r][1], v[r][1]);
                    const bool rowin = kin && in_j[r];
                    nv[r][0] = (rowin && in_i[0]) ? o0 : cc0;
                    nv[r][1] = (rowin && in_i[1]) ? o1 : cc1;
                }
            } else {
#pragma unroll
                for (int r = 0; r < RJ; ++r) nv[r][0] = nv[r][1] = 0.0;
            }
            if (L < T) {
                if (act) {
                    double* dst = lvl + size_t((L - 1) * 2 + (consumed & 1)) * PSTRIDE;
#pragma unroll
                    for (int r = 0; r < RJ; ++r)
                        *reinterpret_cast<double2*>(dst + (r0 + r) * BW + c0) =
                            make_double2(nv[r][0], nv[r][1]);
                }
            } else if (n >= 2 * T) {
                // output tile cells: i - I0 in [0, TI), j - J0 in [0, TJ)
                double* ob = outb + size_t(consumed & 1) * ((C::OUT + 15) / 16 * 16);
                if (di >= 0 && di < C::TO) {
#pragma unroll
                    for (int r = 0; r < RJ; ++r) {
                        const int jj = dj + r;
                        if (jj >= 0 && jj < TJ)
                            *reinterpret_cast<double2*>(ob + jj * C::TO + di) =
                                make_double2(nv[r][0], nv[r][1]);
                    }
                }
            }
            // shift the level-(L-1) z-queue: D <- C <- (value at plane k+1)
#pragma unroll
            for (int r = 0; r < RJ; ++r) {
                qD[L - 1][r][0] = qC[L - 1][r][0];
                qD[L - 1][r][1] = qC[L - 1][r][1];
                qC[L - 1][r][0] = v[r][0];
                qC[L - 1][r][1] = v[r][1];
                v[r][0] = nv[r][0];
                v[r][1] = nv[r][1];
            }
        }
        if (n >= 2 * T) fence_proxy_async_smem();
        if (tid == 0) bulk_wait_read<0>();  // the previous output store has left smem
        __syncthreads();

        if (tid == 0) {
            if (n >= 2 * T) {
                const double* ob = outb + size_t(consumed & 1) * ((C::OUT + 15) / 16 * 16);
                tma_store_3d(&dst_map, ob, it.I0, it.J0, pplane - T);
                bulk_commit();
            }
            // refill the slot freed by this step (plane p_n - 1)
            if (pitem.N > 0) {
                uint64_t* bar = &full[ld_issued % S];
                mbar_arrive_expect_tx(bar, C::BOX_BYTES);
                tma_load_3d(ring + size_t(ld_issued % S) * PSTRIDE, &src_map, pitem.I0 - C::H,
                            pitem.J0 - T, pitem.kb - T + pn, bar);
                ++ld_issued;
                if (++pn == pitem.N) {
                    pn = 0;
                    pq = (pq + 1) % C::QSLOTS;
                    pitem = decode_item<C>(p, atomicAdd(p.counter, 1));
                    queue[pq] = pitem;
                }
            }
        }
        ++consumed;
        if (++n == it.N) {
            n = 0;
            // the producer wrote the next item before issuing its first load,
            // which happened at least one barrier ago
            __syncthreads();
            cq = (cq + 1) % C::QSLOTS;
            it = queue[cq];
        }
    }
    if (tid == 0) bulk_wait<0>();
}

}  // namespace sb
