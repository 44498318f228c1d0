// sb_api.cu -- C ABI (include/stencil_b200.h) over the sm_100a kernels.
//
// Host-side responsibilities: argument validation (mirroring the reference's
// PlanError/PartitionError/DimensionError checks, raised before any work),
// TMA descriptor construction, kernel selection per temporal depth,
// persistent-grid sizing from the SM count, the Dirichlet-halo copy into the
// scratch buffer, and the host-buffer entry point used by the Python drop-in.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdarg>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <climits>
#include <map>
#include <mutex>
#include <queue>
#include <tuple>
#include <string>
#include <vector>

#include "../../include/stencil_b200.h"
#include "jacobi_tb.cuh"
#include "sb_internal.h"

namespace sb {

// ---------------------------------------------------------------------------
// error state
static thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

int cuda_fail(cudaError_t e, const char* what) {
    return fail(SB_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
}

void clear_error() { g_err.clear(); }
const char* last_error() { return g_err.c_str(); }

// ---------------------------------------------------------------------------
// driver entry point for cuTensorMapEncodeTiled (no -lcuda link dependency)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

// 3-D map over a padded grid with a (bw, bh, bd) box; rows `pitch` doubles
// apart (pitch >= nip, even: TMA needs 16-byte row strides).
int make_grid_map3p(CUtensorMap* m, const double* base, int64_t nip, int64_t njp, int64_t nkp,
                    int bw, int bh, int bd, int64_t pitch) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return fail(SB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[3] = {(cuuint64_t)nip, (cuuint64_t)njp, (cuuint64_t)nkp};
    cuuint64_t strides[2] = {(cuuint64_t)(pitch * 8), (cuuint64_t)(pitch * njp * 8)};
    cuuint32_t box[3] = {(cuuint32_t)bw, (cuuint32_t)bh, (cuuint32_t)bd};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides,
                    box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(SB_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return SB_OK;
}

int make_grid_map3(CUtensorMap* m, const double* base, int64_t nip, int64_t njp, int64_t nkp,
                   int bw, int bh, int bd) {
    return make_grid_map3p(m, base, nip, njp, nkp, bw, bh, bd, nip);
}

int make_grid_map(CUtensorMap* m, const double* base, int64_t nip, int64_t njp, int64_t nkp,
                  int bw, int bh) {
    return make_grid_map3(m, base, nip, njp, nkp, bw, bh, 1);
}

// ---------------------------------------------------------------------------
// per-device context: SM count, work counters
// Work counters: every launch takes its own slot from a rotating pool, so
// kernels running concurrently on different streams of one device (z-slabs
// sharing a GPU) never share a counter.
constexpr int kCounterSlots = 4096;
struct DevCtx {
    int sms = 0;
    int* counters = nullptr;  // device ints, kCounterSlots of them
    unsigned seq = 0;         // next slot
};
static std::mutex g_ctx_mu;
static std::vector<DevCtx> g_ctx;

int dev_ctx(DevCtx** out) {
    int dev;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    std::lock_guard<std::mutex> lk(g_ctx_mu);
    if ((int)g_ctx.size() <= dev) g_ctx.resize(dev + 1);
    DevCtx& c = g_ctx[dev];
    if (!c.counters) {
        e = cudaDeviceGetAttribute(&c.sms, cudaDevAttrMultiProcessorCount, dev);
        if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");
        e = cudaMalloc(&c.counters, kCounterSlots * sizeof(int));
        if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(counters)");
    }
    *out = &c;
    return SB_OK;
}

int ctas_per_sm(const void* kern, int threads, size_t smem, int* out) {
    int dev;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, int> known;
    std::lock_guard<std::mutex> lk(mu);
    auto it = known.find({kern, dev});
    if (it != known.end()) {
        *out = it->second;
        return SB_OK;
    }
    if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) !=
        cudaSuccess)
        return cuda_fail(e, "cudaFuncSetAttribute");
    int o = 0;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, threads, smem)) != cudaSuccess)
        return cuda_fail(e, "occupancy query");
    if (o < 1) return fail(SB_ERR_CUDA, "kernel does not fit on an SM (%zu B shared memory)", smem);
    known[{kern, dev}] = o;
    *out = o;
    return SB_OK;
}

int get_counters(int** counters, int* sms) {
    DevCtx* c;
    int rc = dev_ctx(&c);
    if (rc) return rc;
    std::lock_guard<std::mutex> lk(g_ctx_mu);
    *counters = c->counters + (c->seq++ % kCounterSlots);
    *sms = c->sms;
    return SB_OK;
}

// ---------------------------------------------------------------------------
// kernels: halo copy and the generic (odd pitch) Jacobi sweep

// Copies every halo (Dirichlet) cell of src into dst.
__global__ void halo_copy_kernel(const double* __restrict__ src, double* __restrict__ dst, int ni,
                                 int nj, int nk) {
    const int64_t nip = ni + 2, njp = nj + 2, plane = nip * njp;
    // faces: k = 0 and k = nk+1 planes (full), then per interior plane the
    // j = 0 / nj+1 rows and the i = 0 / ni+1 columns
    const int64_t n_kfaces = 2 * plane;
    const int64_t n_rows = (int64_t)nk * 2 * nip;
    const int64_t n_cols = (int64_t)nk * nj * 2;
    const int64_t total = n_kfaces + n_rows + n_cols;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t off;
        if (t < n_kfaces) {
            off = (t < plane) ? t : (int64_t)(nk + 1) * plane + (t - plane);
        } else if (t < n_kfaces + n_rows) {
            int64_t u = t - n_kfaces;
            int64_t k = 1 + u / (2 * nip), r = u % (2 * nip);
            int64_t j = (r < nip) ? 0 : nj + 1, i = r % nip;
            off = k * plane + j * nip + i;
        } else {
            int64_t u = t - n_kfaces - n_rows;
            int64_t k = 1 + u / (2 * nj), r = u % (2 * nj);
            int64_t j = 1 + r / 2, i = (r & 1) ? ni + 1 : 0;
            off = k * plane + j * nip + i;
        }
        dst[off] = src[off];
    }
}

// One plain sweep for grids whose row pitch is not a 16-byte multiple (odd
// ni), where TMA cannot describe the grid.  Thread per (i, j) column,
// register z-queue, neighbours through the read-only path.
__global__ void jacobi_generic_kernel(const double* __restrict__ src, double* __restrict__ dst,
                                      int ni, int nj, int kfirst, int klast, int kchunk, double a,
                                      double b) {
    const int i = 1 + blockIdx.x * blockDim.x + threadIdx.x;
    const int j = 1 + blockIdx.y * blockDim.y + threadIdx.y;
    if (i > ni || j > nj) return;
    const int64_t nip = ni + 2, plane = nip * (nj + 2);
    const int k0 = kfirst + blockIdx.z * kchunk, k1 = min(k0 + kchunk, klast);
    const double* s = src + j * nip + i;
    double d = __ldg(s + (k0 - 1) * plane), c = __ldg(s + k0 * plane);
    for (int k = k0; k < k1; ++k) {
        const double* q = s + k * plane;
        const double u = __ldg(q + plane);
        dst[k * plane + j * nip + i] =
            jac_cell(a, b, c, __ldg(q - 1), __ldg(q + 1), __ldg(q - nip), __ldg(q + nip), d, u);
        d = c;
        c = u;
    }
}

// STREAM-style triad a[i] = b[i] + s*c[i] (reference perf.py:45-48, the
// bandwidth probe behind predict_p0): 16-byte vector accesses, grid-stride,
// no contraction (bitwise equal to the numpy check of the reference).
__global__ void triad_kernel(double* __restrict__ a, const double* __restrict__ b,
                             const double* __restrict__ c, double s, int64_t n) {
    const int64_t n2 = n / 2;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n2; t += stride) {
        const double2 x = reinterpret_cast<const double2*>(b)[t];
        const double2 y = reinterpret_cast<const double2*>(c)[t];
        reinterpret_cast<double2*>(a)[t] =
            make_double2(__dadd_rn(x.x, __dmul_rn(s, y.x)), __dadd_rn(x.y, __dmul_rn(s, y.y)));
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) a[n - 1] = __dadd_rn(b[n - 1], __dmul_rn(s, c[n - 1]));
}

// FP64 pipe probe: kFp64Chains independent DADD chains per thread, no memory
// traffic in the loop.  With the SMs full of warps this runs at the FP64
// pipe's issue limit: the secondary ceiling of the stencil kernels (SURVEY
// 8(d): "fp64 pipe ... measure on the box").
constexpr int kFp64Chains = 8;
__global__ void fp64_probe_kernel(double* sink, int64_t iters) {
    double x[kFp64Chains];
#pragma unroll
    for (int c = 0; c < kFp64Chains; ++c) x[c] = 1.0 + 1e-3 * (threadIdx.x + c);
    const double d = 1e-300 * (1 + blockIdx.x % 3);
    for (int64_t i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < kFp64Chains; ++c) x[c] = __dadd_rn(x[c], d);
    }
    double acc = 0;
#pragma unroll
    for (int c = 0; c < kFp64Chains; ++c) acc = __dadd_rn(acc, x[c]);
    if (acc == 12345.0) sink[threadIdx.x] = acc;  // keeps the chains alive
}

// ---------------------------------------------------------------------------
// temporally blocked launch

// Per tile: 1 if the tile's computed region touches the i/j boundary (its
// interior steps run in MASK mode; jacobi_tb.cuh, the kernel's ij_in).
template <class C>
static std::vector<char> border_tiles(int ni, int nj, int tiles_i, int tiles_j) {
    std::vector<char> v(size_t(tiles_i) * tiles_j);
    for (int tj = 0; tj < tiles_j; ++tj)
        for (int ti = 0; ti < tiles_i; ++ti) {
            const int I0 = C::TO * ti, jlo = 1 + C::TJ * tj - (C::T - 1);
            const bool in = (I0 - C::H >= 1) && (I0 - C::H + C::BW - 1 <= ni) && (jlo >= 1) &&
                            (jlo + C::ROWS - 1 <= nj);
            v[size_t(tj) * tiles_i + ti] = in ? 0 : 1;
        }
    return v;
}

// Tile grid and k-block length of one launch (shared by the launch and the
// schedule query sb_jacobi_schedule, so both see the same decomposition).
struct TbPlan {
    int tiles_i, tiles_j, kb;
    bool list_ok;  // explicit item list allowed (not overridden by SB_KBLK)
};

template <class C>
static TbPlan tb_plan(int ni, int nj, int kfirst, int klast, int grid) {
    TbPlan pl;
    pl.tiles_i = (ni + 1 + C::TO - 1) / C::TO;  // tiles [TO*t, TO*t+TO) must cover [1, ni]
    pl.tiles_j = (nj + C::TJ - 1) / C::TJ;
    const int nkout = klast - kfirst;
    int kb = pick_kblock(C::T, pl.tiles_i * pl.tiles_j, nkout, grid);
    static const int kb_env = tune_env("SB_KBLK") ? atoi(tune_env("SB_KBLK")) : 0;  // tuning
    if (kb_env > 0) kb = kb_env;
    pl.kb = std::max(1, std::min(kb, nkout));
    pl.list_ok = kb_env <= 0;
    return pl;
}

template <class C, bool AZ>
static int launch_tb_impl(const double* src, double* dst, int ni, int nj, int nk, int kfirst,
                          int klast, double a, double b, cudaStream_t st, int64_t pitch,
                          const JacPeers* peers) {
    int* counters;
    int sms;
    int rc = get_counters(&counters, &sms);
    if (rc) return rc;
    // the fused-exchange variant only where a launch sends planes
    auto kern = peers ? jacobi_tb_kernel<C, AZ, true> : jacobi_tb_kernel<C, AZ, false>;
    int per_sm = 0;
    if ((rc = ctas_per_sm((const void*)kern, C::NT, C::SMEM_BYTES, &per_sm))) return rc;
    const int occ = per_sm * sms;  // resident CTAs on the device
    CUtensorMap smap, dmap;
    const int64_t nip = ni + 2, njp = nj + 2, nkp = nk + 2;
    if (pitch <= 0) pitch = nip;
    // without TS the kernel addresses dst directly with the dense pitch
    if (!C::TS && pitch != nip) return fail(SB_ERR_PLAN, "pitched grids need a TMA-store depth");
    if ((rc = make_grid_map3p(&smap, src, nip, njp, nkp, C::BW, C::BH, 1, pitch))) return rc;
    if (C::TS) {
        if ((rc = make_grid_map3p(&dmap, dst, nip, njp, nkp, C::TO, C::TJ, 1, pitch))) return rc;
    } else {
        dmap = smap;  // unused
    }

    JacobiParams p;
    p.ni = ni;
    p.nj = nj;
    p.nk = nk;
    memset(&p.peers, 0, sizeof p.peers);
    if (peers) {
        if (!C::TS || pitch != nip) return fail(SB_ERR_PLAN, "fused halo exchange needs a TMA-store depth");
        p.peers = *peers;
    }
    const int grid = occ;  // resident CTAs
    const TbPlan pl = tb_plan<C>(ni, nj, kfirst, klast, grid);
    p.tiles_i = pl.tiles_i;
    p.tiles_j = pl.tiles_j;
    const int tiles = p.tiles_i * p.tiles_j;
    const int nkout = klast - kfirst;
    const int kb = pl.kb;
    p.kfirst = kfirst;
    p.klast = klast;
    p.kblk = kb;
    p.kblocks = (nkout + kb - 1) / kb;
    p.items = tiles * p.kblocks;
    p.list = nullptr;
    if (C::T >= 3) {  // explicit item list (always: these kernels decode no other form)
        const int4* list;
        int count;
        if ((rc = item_list(C::T, p.tiles_i, p.tiles_j, border_tiles<C>(ni, nj, p.tiles_i, p.tiles_j),
                            kfirst, klast, grid, kb, !pl.list_ok, &list, &count)))
            return rc;
        if (!list) return fail(SB_ERR_PLAN, "no item list for depth %d", C::T);
        p.list = list;
        p.items = count;
    }
    p.a = a;
    p.b = b;
    p.counter = counters;
    p.dst = dst;
    p.plane = nip * njp;
    cudaError_t e = cudaMemsetAsync(counters, 0, sizeof(int), st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(counter)");
    kern<<<min(grid, p.items), C::NT, C::SMEM_BYTES, st>>>(smap, dmap, p);
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "jacobi_tb launch");
    return SB_OK;
}


template <class C>
static int launch_tb(const double* src, double* dst, int ni, int nj, int nk, int kfirst, int klast,
                     double a, double b, cudaStream_t st, int64_t pitch = 0,
                     const JacPeers* peers = nullptr) {
    if (a == 0.0)
        return launch_tb_impl<C, true>(src, dst, ni, nj, nk, kfirst, klast, a, b, st, pitch, peers);
    return launch_tb_impl<C, false>(src, dst, ni, nj, nk, kfirst, klast, a, b, st, pitch, peers);
}

// Tile configurations per depth: <T, RJ rows/thread, NW warps, S ring stages,
// MINB, L1S level 1 from the ring, TS TMA-store output>.
// Builds with -DSB_EXPERIMENTS (tools/, never the product library) also carry
// the alternatives measured while tuning, selected with SB_JCFG=<variant>.
#ifdef SB_EXPERIMENTS
static int jcfg_variant() {
    static int v = getenv("SB_JCFG") ? atoi(getenv("SB_JCFG")) : 0;
    return v;
}
#endif

// Calls f(JacobiCfg<...>{}) with the tile configuration of depth T.
template <class F>
static int with_cfg(int T, F&& f) {
#define SB_L(...) return f(JacobiCfg<__VA_ARGS__>{})
#ifdef SB_EXPERIMENTS
    const int v = jcfg_variant();
    switch (T) {
        case 3:
            if (v == 7) SB_L(3, 5, 8, 6, 1, false, true);
            if (v == 10) SB_L(3, 4, 8, 8, 1, false, true, true);
            if (v == 11) SB_L(3, 5, 8, 6, 1, false, true, true);
            if (v == 12) SB_L(3, 6, 8, 5, 1, false, true, true);
            if (v == 13) SB_L(3, 6, 8, 5, 1, false, true);
            if (v == 14) SB_L(3, 5, 8, 7, 1, false, true);
            if (v == 16) SB_L(3, 6, 8, 6, 1, false, true);
            if (v == 17) SB_L(3, 6, 8, 4, 1, false, true);
            break;
        case 4:
            if (v == 10) SB_L(4, 4, 8, 8, 1, false, true, true);
            if (v == 11) SB_L(4, 5, 8, 6, 1, false, true, true);
            if (v == 12) SB_L(4, 5, 8, 5, 1, false, true, true);
            if (v == 15) SB_L(4, 5, 8, 6, 1, true, true);
            break;
        case 2:
            if (v == 20) SB_L(2, 6, 8, 6, 1, false, true);
            if (v == 21) SB_L(2, 8, 8, 4, 1, false, true);
            if (v == 23) SB_L(2, 6, 8, 5, 1, false, true);
            break;
    }
#endif
    switch (T) {
        case 1: SB_L(1, 4, 8, 4, 2, false, true);
        // T = 2, 3: 6 rows per thread (64 x 48 tiles) -- registers allow it at
        // these depths; taller tiles cut the j-overlap (round 2: T=2 647 -> 709
        // GLUP/s at 1024^3, 663 -> 730 at 512^3; T=3 783 -> 845, 717 -> 808;
        // profiles/r2/ab_t2_t3_tall_tiles.log)
        case 2: SB_L(2, 6, 8, 6, 1, false, true);
        case 3: SB_L(3, 6, 8, 5, 1, false, true);
        case 4: SB_L(4, 4, 8, 8, 1, false, true);
        // depths 5-8 (the slab path's ghost-zone blocks, the config-3 "steps
        // per HBM pass" sweep): 12 warps x 2 rows; level 1 reads the TMA
        // ring (L1S), level T stores through TMA (TS), one step loop (UNI) --
        // the register-lean form (ptxas: 0 / 0 / 12 / 952 spill bytes at
        // T = 5..8; the plain form spilled 0 / 156 / 6364 / 9736).  Every
        // depth stores through TMA, which the fused slab exchange relies on.
        case 5: SB_L(5, 2, 12, 3, 1, true, true);
        case 6: SB_L(6, 2, 12, 3, 1, true, true, true);
        case 7: SB_L(7, 2, 12, 3, 1, true, true, true);
        case 8: SB_L(8, 2, 12, 3, 1, true, true, true);
    }
#undef SB_L
    return fail(SB_ERR_PLAN, "unsupported depth %d", T);
}

static int launch_depth(int T, const double* src, double* dst, int ni, int nj, int nk, int kfirst,
                        int klast, double a, double b, cudaStream_t st, int64_t pitch = 0,
                        const JacPeers* peers = nullptr) {
    if (klast <= kfirst) return SB_OK;
    return with_cfg(T, [&](auto cfg) {
        return launch_tb<decltype(cfg)>(src, dst, ni, nj, nk, kfirst, klast, a, b, st, pitch, peers);
    });
}

// The work items of one launch (see sb_jacobi_schedule).
template <class C>
static int schedule_query(int ni, int nj, int kfirst, int klast, int ctas, int32_t* items,
                          int64_t cap, int64_t* count, int32_t* dims) {
    const TbPlan pl = tb_plan<C>(ni, nj, kfirst, klast, ctas);
    std::vector<int4> v;
    if (pl.list_ok)
        v = build_item_list(C::T, pl.tiles_i, pl.tiles_j,
                            border_tiles<C>(ni, nj, pl.tiles_i, pl.tiles_j), kfirst, klast, ctas,
                            pl.kb);
    if (v.empty())  // the regular decomposition, in claim order (k-block major)
        for (int k0 = kfirst; k0 < klast; k0 += pl.kb)
            for (int t = 0; t < pl.tiles_i * pl.tiles_j; ++t)
                v.push_back(make_int4(t, k0, std::min(k0 + pl.kb, klast), 0));
    if (dims) {
        dims[0] = C::TO;
        dims[1] = C::TJ;
        dims[2] = pl.tiles_i;
        dims[3] = pl.tiles_j;
    }
    *count = (int64_t)v.size();
    for (int64_t x = 0; x < std::min<int64_t>(cap, (int64_t)v.size()); ++x) {
        items[4 * x + 0] = v[x].x % pl.tiles_i;
        items[4 * x + 1] = v[x].x / pl.tiles_i;
        items[4 * x + 2] = v[x].y;
        items[4 * x + 3] = v[x].z;
    }
    return SB_OK;
}

static int launch_generic(const double* src, double* dst, int ni, int nj, int kfirst, int klast,
                          double a, double b, cudaStream_t st) {
    if (klast <= kfirst) return SB_OK;
    dim3 blk(32, 8);
    const int kchunk = 64;
    dim3 grd((ni + 31) / 32, (nj + 7) / 8, (klast - kfirst + kchunk - 1) / kchunk);
    jacobi_generic_kernel<<<grd, blk, 0, st>>>(src, dst, ni, nj, kfirst, klast, kchunk, a, b);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? SB_OK : cuda_fail(e, "jacobi_generic launch");
}

int jacobi_generic_sweep(const double* src, double* dst, int ni, int nj, int nk, double a, double b,
                         cudaStream_t st) {
    return launch_generic(src, dst, ni, nj, 1, nk + 1, a, b, st);
}

int check_dims(int64_t ni, int64_t nj, int64_t nk) {
    if (ni < 1 || nj < 1 || nk < 1)
        return fail(SB_ERR_DIMENSION, "extents must be positive, got %lldx%lldx%lld",
                    (long long)ni, (long long)nj, (long long)nk);
    // int32 indexing inside kernels and TMA coordinates
    // (plane offsets are 32-bit: (ni+2)(nj+2) < 2^31)
    if (ni > (1 << 20) || nj > (1 << 20) || nk > (1 << 20) ||
        (ni + 2) * (nj + 2) >= (int64_t(1) << 31) ||
        (ni + 2) * (nj + 2) * (nk + 2) > (int64_t(1) << 40))
        return fail(SB_ERR_DIMENSION, "grid %lldx%lldx%lld too large", (long long)ni,
                    (long long)nj, (long long)nk);
    return SB_OK;
}

bool tma_ok(const void* p, int64_t ni) {
    return ((ni + 2) % 2 == 0) && ((reinterpret_cast<uintptr_t>(p) & 15) == 0);
}

int halo_copy(const double* src, double* dst, int ni, int nj, int nk, cudaStream_t st) {
    halo_copy_kernel<<<256, 256, 0, st>>>(src, dst, ni, nj, nk);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? SB_OK : cuda_fail(e, "halo_copy launch");
}

// T fused sweeps src -> dst (T = 1 for grids TMA cannot describe), output
// planes [kfirst, klast) only.
int jacobi_block(const double* src, double* dst, int ni, int nj, int nk, int kfirst, int klast,
                 int T, double a, double b, cudaStream_t st, const JacPeers* peers) {
    if (peers) {  // fused exchange: the TMA path only (the caller checked tma_ok)
        if (!(tma_ok(src, ni) && tma_ok(dst, ni))) return fail(SB_ERR_PLAN, "fused exchange needs even ni");
        return launch_depth(T, src, dst, ni, nj, nk, kfirst, klast, a, b, st, 0, peers);
    }
    if (tma_ok(src, ni) && tma_ok(dst, ni))
        return launch_depth(T, src, dst, ni, nj, nk, kfirst, klast, a, b, st);
    if (T != 1) return fail(SB_ERR_PLAN, "depth %d needs an even ni (16-byte row pitch)", T);
    return launch_generic(src, dst, ni, nj, kfirst, klast, a, b, st);
}

// Deepest fused launch worth running on a full domain: beyond T = 4 the
// trapezoid overlap (and the register queues) cost more than the HBM
// traffic saved, so deeper requests run as back-to-back 4-sweep launches
// (bit-identical: the depth is a schedule, not part of the arithmetic).
constexpr int kMaxFusedDepth = 4;

// Advance `iters` Jacobi sweeps between two device buffers whose halos are
// already equal.  Returns through *in_b whether the result is in `b_buf`.
// Grids TMA cannot describe directly (odd ni, or buffers not 16-byte
// aligned) that are worth it run the fused kernel on pitched copies: rows
// padded to an even number of doubles (outside the tensor maps' extent, so
// never touched), copied in with cudaMemcpy2D and the result copied back
// into a_buf.  Two scratch buffers per device, grown on demand.
// Calls on two streams of one device are serialised through `last`.
struct JacPitched {
    double* buf[2] = {nullptr, nullptr};
    size_t cap = 0;  // doubles per buffer
    cudaEvent_t last = nullptr;  // after the previous user's copy-out (any stream)
};
static JacPitched g_jac_pitched[64];
static std::mutex g_jac_pitched_mu;

// frees the pitched-copy buffers of `dev` (caller synchronised the device);
// true if there were any
bool jacobi_release(int dev) {
    if (dev < 0 || dev >= 64) return false;
    std::lock_guard<std::mutex> lk(g_jac_pitched_mu);
    bool had = false;
    for (double*& q : g_jac_pitched[dev].buf) {
        had = had || q;
        if (q) cudaFree(q);
        q = nullptr;
    }
    g_jac_pitched[dev].cap = 0;
    return had;
}

bool jacobi_holds(int dev) {
    if (dev < 0 || dev >= 64) return false;
    std::lock_guard<std::mutex> lk(g_jac_pitched_mu);
    return g_jac_pitched[dev].buf[0] != nullptr;
}

static int jacobi_run_pitched(double* a_buf, int ni, int nj, int nk, int64_t iters, double a,
                              double b, int depth, cudaStream_t st) {
    int dev;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    if (dev >= 64) return fail(SB_ERR_CUDA, "device index %d unsupported", dev);
    std::lock_guard<std::mutex> lk(g_jac_pitched_mu);
    JacPitched& P = g_jac_pitched[dev];
    if (!P.last && (e = cudaEventCreateWithFlags(&P.last, cudaEventDisableTiming)) != cudaSuccess)
        return cuda_fail(e, "cudaEventCreate");
    if ((e = cudaStreamWaitEvent(st, P.last, 0)) != cudaSuccess) return cuda_fail(e, "cudaStreamWaitEvent");
    const int64_t nip = ni + 2, pitch = (nip + 1) / 2 * 2, rows = int64_t(nj + 2) * (nk + 2);
    const size_t need = size_t(pitch) * size_t(rows);
    if (P.cap < need) {
        if ((P.buf[0] || P.buf[1]) && (e = cudaStreamSynchronize(st)) != cudaSuccess)
            return cuda_fail(e, "sync");
        for (double*& q : P.buf) {
            if (q) cudaFree(q);
            q = nullptr;
        }
        P.cap = 0;
        for (double*& q : P.buf)
            if ((e = cudaMalloc(&q, need * sizeof(double))) != cudaSuccess)
                return cuda_fail(e, "cudaMalloc(pitched Jacobi grid)");
        P.cap = need;
    }
    for (double* q : P.buf)  // both copies carry the Dirichlet halo
        if ((e = cudaMemcpy2DAsync(q, pitch * 8, a_buf, nip * 8, nip * 8, rows,
                                   cudaMemcpyDeviceToDevice, st)) != cudaSuccess)
            return cuda_fail(e, "cudaMemcpy2DAsync(in)");
    double* src = P.buf[0];
    double* dst = P.buf[1];
    for (int64_t left = iters; left > 0;) {
        const int T = (int)std::min<int64_t>(left, depth);
        int rc = launch_depth(T, src, dst, ni, nj, nk, 1, nk + 1, a, b, st, pitch);
        if (rc) return rc;
        left -= T;
        std::swap(src, dst);
    }
    if ((e = cudaMemcpy2DAsync(a_buf, nip * 8, src, pitch * 8, nip * 8, rows,
                               cudaMemcpyDeviceToDevice, st)) != cudaSuccess)
        return cuda_fail(e, "cudaMemcpy2DAsync(out)");
    if ((e = cudaEventRecord(P.last, st)) != cudaSuccess) return cuda_fail(e, "cudaEventRecord");
    return SB_OK;
}

int jacobi_run(double* a_buf, double* b_buf, int ni, int nj, int nk, int64_t iters, double a,
               double b, int depth, cudaStream_t st, int* in_b) {
    const bool tma = tma_ok(a_buf, ni) && tma_ok(b_buf, ni);
    depth = std::min(depth, kMaxFusedDepth);
    if (!tma && depth > 1 && int64_t(ni) * nj * nk * iters >= (int64_t(1) << 22)) {
        *in_b = 0;
        return jacobi_run_pitched(a_buf, ni, nj, nk, iters, a, b, depth, st);
    }
    double* src = a_buf;
    double* dst = b_buf;
    int64_t left = iters;
    while (left > 0) {
        int T = (int)((left >= depth) ? depth : left);
        if (!tma) T = 1;
        int rc = jacobi_block(src, dst, ni, nj, nk, 1, nk + 1, T, a, b, st);
        if (rc) return rc;
        left -= T;
        double* t = src;
        src = dst;
        dst = t;
    }
    *in_b = (src == b_buf);
    return SB_OK;
}

}  // namespace sb

using namespace sb;

extern "C" {

int sb_version(void) { return 100; }

const char* sb_last_error(void) { return sb::last_error(); }

int sb_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int sb_max_depth(void) { return 8; }

int sb_jacobi_schedule(int sweeps, int64_t ni, int64_t nj, int64_t k_out_lo, int64_t k_out_hi,
                       int ctas, int32_t* items, int64_t cap, int64_t* count, int32_t* dims) {
    clear_error();
    int rc = check_dims(ni, nj, std::max<int64_t>(1, k_out_hi));
    if (rc) return rc;
    if (sweeps < 1 || sweeps > sb_max_depth())
        return fail(SB_ERR_PLAN, "sweeps per block must be in [1, %d], got %d", sb_max_depth(), sweeps);
    if (ni % 2) return fail(SB_ERR_PLAN, "odd ni runs the generic sweep kernel (no tiled items)");
    if (k_out_lo < 1 || k_out_hi <= k_out_lo)
        return fail(SB_ERR_ARGUMENT, "bad plane range [%lld, %lld)", (long long)k_out_lo,
                    (long long)k_out_hi);
    if (ctas < 1) return fail(SB_ERR_ARGUMENT, "ctas must be >= 1");
    if (!count || (cap > 0 && !items)) return fail(SB_ERR_ARGUMENT, "null pointer");
    return with_cfg(sweeps, [&](auto cfg) {
        return schedule_query<decltype(cfg)>((int)ni, (int)nj, (int)k_out_lo, (int)k_out_hi, ctas,
                                             items, cap, count, dims);
    });
}

int sb_jacobi(double* grid, double* scratch, int64_t ni, int64_t nj, int64_t nk, int64_t iters,
              double a, double b, int depth, void* stream, int* result_in_scratch) {
    clear_error();
    int rc = check_dims(ni, nj, nk);
    if (rc) return rc;
    if (iters < 0) return fail(SB_ERR_PLAN, "iter_end must be >= 0, got %lld", (long long)iters);
    if (depth < 1 || depth > sb_max_depth())
        return fail(SB_ERR_PLAN, "depth must be in [1, %d], got %d", sb_max_depth(), depth);
    if (!grid || !scratch || !result_in_scratch) return fail(SB_ERR_ARGUMENT, "null pointer");
    if (grid == scratch) return fail(SB_ERR_ARGUMENT, "grid and scratch must be distinct");
    if ((reinterpret_cast<uintptr_t>(grid) | reinterpret_cast<uintptr_t>(scratch)) & 7)
        return fail(SB_ERR_ARGUMENT, "grid buffers must be 8-byte aligned");
    *result_in_scratch = 0;
    if (iters == 0) return SB_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if ((rc = halo_copy(grid, scratch, (int)ni, (int)nj, (int)nk, st))) return rc;
    return jacobi_run(grid, scratch, (int)ni, (int)nj, (int)nk, iters, a, b, depth, st,
                      result_in_scratch);
}

int sb_triad(double* a, const double* b, const double* c, double s, int64_t n, void* stream) {
    clear_error();
    if (n < 0) return fail(SB_ERR_ARGUMENT, "negative element count");
    if (n == 0) return SB_OK;
    if (!a || !b || !c) return fail(SB_ERR_ARGUMENT, "null pointer");
    if ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b) | reinterpret_cast<uintptr_t>(c)) & 15)
        return fail(SB_ERR_ARGUMENT, "triad arrays must be 16-byte aligned");
    int* counters;
    int sms;
    int rc = get_counters(&counters, &sms);
    if (rc) return rc;
    triad_kernel<<<sms * 8, 256, 0, static_cast<cudaStream_t>(stream)>>>(a, b, c, s, n);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? SB_OK : cuda_fail(e, "triad launch");
}

int sb_fp64_probe(double* sink, int64_t iters, void* stream, int64_t* ops) {
    clear_error();
    if (!sink || !ops || iters < 1) return fail(SB_ERR_ARGUMENT, "need a sink, an op counter and iters >= 1");
    int dev = 0, sms = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return cuda_fail(e, "device query");
    const int blocks = sms * 8, threads = 256;  // 64 warps per SM
    fp64_probe_kernel<<<blocks, threads, 0, static_cast<cudaStream_t>(stream)>>>(sink, iters);
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "fp64 probe launch");
    *ops = int64_t(blocks) * threads * iters * kFp64Chains;
    return SB_OK;
}

double* sb_host_alloc(int64_t count) {
    clear_error();
    void* p = nullptr;
    if (count <= 0) return nullptr;
    cudaError_t e = cudaMallocHost(&p, (size_t)count * sizeof(double));
    if (e != cudaSuccess) {
        cuda_fail(e, "cudaMallocHost");
        return nullptr;
    }
    return static_cast<double*>(p);
}

void sb_host_free(double* p) {
    if (p) cudaFreeHost(p);
}

}  // extern "C"
