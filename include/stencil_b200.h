/*
 * stencil_b200.h -- C ABI of the B200-native stencil sweep library
 * (paper_1004_1741_b200/libsb200.so).
 *
 * Drop-in boundary for the reference package `stencilbench`
 * (arxiv 1004.1741).  The reference has no FFI of its own: its hot path is
 * the Python entry `sweeps.run(plan, g)` (pkg/src/stencilbench/sweeps/
 * __init__.py:52-71) dispatching to engines that call numba plane-window
 * kernels.  Each entry point below replaces one engine (see INTEGRATION.md
 * for the ctypes binding a maintainer adds on the reference side):
 *
 *   sb_jacobi / sb_run_host(JACOBI)  <- run_serial / run_threaded_jacobi /
 *                                       run_wavefront_jacobi
 *                                       (sweeps/serial.py:8-42,
 *                                        sweeps/threaded.py:28-59,
 *                                        sweeps/wavefront.py:133-137,160-312)
 *   sb_gs / sb_run_host(GS_*)        <- run_serial / run_pipeline_gs /
 *                                       run_wavefront_gs (GS kernels)
 *                                       (sweeps/threaded.py:62-96,
 *                                        sweeps/wavefront.py:139-143,315-376)
 *   sb_jacobi_slabs / sb_jacobi_planes / sb_slab_layout
 *                                    <- run_threaded_jacobi's k-slab split
 *                                       (sweeps/threaded.py:28-59, :39)
 *                                       across GPUs (z-slabs + halo exchange)
 *   sb_gs_slabs / sb_gs_slab_layout  <- run_pipeline_gs's pipelined order
 *                                       (sweeps/threaded.py:62-96) as a
 *                                       cross-GPU z-pipeline of slabs
 *
 * Grid layout (reference grid.py:61-91): (nk+2) x (nj+2) x (ni+2) doubles,
 * C order, i unit stride; interior cell (k,j,i) at padded (k+1,j+1,i+1);
 * halo cells are Dirichlet data and are never written.
 *
 * Arithmetic (reference kernels.py:125-187): bitwise identical to the
 * reference for every entry point and every depth --
 *   Jacobi:          a*c + b*(((((W+E)+S)+N)+D)+U)
 *   GS naive:        b*(((((W+E)+S)+N)+D)+U)            in lexicographic order
 *   GS interleaved:  b*(W + ((((E+S)+N)+D)+U))          in lexicographic order
 *
 * Errors: every function returns an sb_status; 0 is success.  Argument
 * errors are detected before any device work (like the reference's
 * PlanError / PartitionError, raised before threads start).  The message of
 * the last error on the calling thread is sb_last_error().
 *
 * Threading: calls are synchronous with respect to `stream` only when the
 * function says so; device-pointer entry points enqueue work on `stream`
 * (a cudaStream_t, NULL = legacy default stream) and return.  Not
 * reentrant across threads for the same buffers.
 */
#ifndef STENCIL_B200_H
#define STENCIL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SB_OK = 0,
    SB_ERR_DIMENSION = 1,  /* -> DimensionError (grid extents)            */
    SB_ERR_PLAN = 2,       /* -> PlanError (iters < 0, bad kernel/depth)   */
    SB_ERR_CONFIG = 3,     /* -> ConfigError                                */
    SB_ERR_PARTITION = 4,  /* -> PartitionError (more slabs than planes)   */
    SB_ERR_CUDA = 5,       /* -> DeviceError (CUDA runtime/launch failure)  */
    SB_ERR_TIMEOUT = 6,    /* -> DeviceError (inter-CTA flag wait expired)  */
    SB_ERR_ARGUMENT = 7,   /* -> ValueError (null/misaligned pointer)       */
    SB_ERR_NODEVICE = 8    /* -> DeviceError (no CUDA device)               */
} sb_status;

typedef enum {
    SB_KERNEL_JACOBI = 0,
    SB_KERNEL_GS_NAIVE = 1,
    SB_KERNEL_GS_INTERLEAVED = 2
} sb_kernel;

/* Library/ABI version (major*10000 + minor*100 + patch). */
int sb_version(void);

/* Message of the last failing call on this thread ("" if none). */
const char* sb_last_error(void);

/* Number of visible CUDA devices (0 when none). */
int sb_device_count(void);

/* Maximum temporal block depth supported by sb_jacobi. */
int sb_max_depth(void);

/*
 * Diagnostic (host only, no GPU work): the work items of one fused launch
 * of `sweeps` (1..sb_max_depth()) Jacobi sweeps writing planes
 * [k_out_lo, k_out_hi) of an ni x nj grid (even ni: the tiled kernel) on a
 * device with `ctas` resident CTAs, in the order the CTAs claim them.  Item
 * x is items[4x..4x+3] = (tile_i, tile_j, k0, k1): output columns
 * [TO*tile_i, TO*tile_i + TO), rows [1 + TJ*tile_j, 1 + TJ*tile_j + TJ),
 * planes [k0, k1).  Writes min(cap, *count) items; dims (may be NULL)
 * receives (TO, TJ, tiles_i, tiles_j).  Every (tile, plane) of the launch
 * appears in exactly one item -- tests/test_lib.py checks that property.
 * No Python-reference counterpart: it exposes the schedule of
 * sb_jacobi / sb_jacobi_planes ("Schedule").
 */
int sb_jacobi_schedule(int sweeps, int64_t ni, int64_t nj, int64_t k_out_lo, int64_t k_out_hi,
                       int ctas, int32_t* items, int64_t cap, int64_t* count, int32_t* dims);

/*
 * Jacobi sweeps on device memory.  `grid` and `scratch` are device
 * pointers to two distinct padded grids; `scratch` needs no initialisation
 * (its halo is copied from `grid` on the stream).  Advances `iters` sweeps,
 * fusing up to `depth` (1..sb_max_depth()) sweeps per HBM pass (depths
 * above 4 run as 4-sweep passes: sustained under the board power cap, 4 is
 * the fastest fused depth on B200; results are identical for every depth);
 * iters that are not a multiple of the pass depth end with a shallower pass.  On return
 * *result_in_scratch tells which buffer holds the final field (the other
 * holds an intermediate one), like run_serial returning the copy for odd
 * iteration counts.  Asynchronous on `stream`.
 */
int sb_jacobi(double* grid, double* scratch, int64_t ni, int64_t nj, int64_t nk,
              int64_t iters, double a, double b, int depth, void* stream,
              int* result_in_scratch);

/*
 * Lexicographic Gauss-Seidel sweeps, in place on the device grid.
 * kernel: SB_KERNEL_GS_NAIVE or SB_KERNEL_GS_INTERLEAVED (selects the
 * association, bitwise equal to the matching reference kernel).
 * Asynchronous on `stream`.  GS calls on one device share its scheduling
 * state; calls on different streams of one device are serialised by the
 * library (each launch waits for the previous one on that device).
 */
int sb_gs(double* grid, int64_t ni, int64_t nj, int64_t nk, int64_t iters, double b,
          int kernel, void* stream);

/*
 * Wait for all work queued on `stream` and report deferred failures: a
 * CUDA error raised by the kernels, or SB_ERR_TIMEOUT when a Gauss-Seidel
 * inter-CTA dependency wait expired.  A timed-out launch is abandoned
 * cooperatively: every warp of every CTA sees the error word and exits, so
 * the CUDA context stays usable (the next call runs normally); the grid
 * content is then unspecified.  This replaces the reference's poisoned
 * barriers (sync.py:31-32) and worker re-raise (sweeps/team.py:42-64).
 */
int sb_sync(void* stream);

/*
 * Test hook (fault injection, used by tests/test_gpu_faults.py): kind 1
 * makes later Gauss-Seidel launches withhold one progress publish (tile 0,
 * sweep 0, chunks after the first), so its dependants wait until the
 * timeout; kind 0 restores normal operation.  timeout_cycles (> 0) sets the
 * no-progress limit of the inter-CTA waits in SM clock cycles; <= 0 restores
 * the default 2^35 (~17 s).  Process-wide; affects launches issued later.
 */
int sb_debug_fault(int kind, int64_t timeout_cycles);

/*
 * The library's plain "serial engine": straightforward kernels without
 * tiling or temporal blocking (one sweep per launch for Jacobi, a single
 * thread in exact lexicographic order for GS).  Used by the CLI's verify to
 * check the optimised paths, as the reference's verify checks its variants
 * against run_serial (cli.py:297-331).  Slow by design.  Jacobi ping-pongs
 * grid/scratch like sb_jacobi; GS ignores scratch and a.  Asynchronous.
 */
int sb_reference_sweeps(int kernel, double* grid, double* scratch, int64_t ni, int64_t nj,
                        int64_t nk, int64_t iters, double a, double b, void* stream,
                        int* result_in_scratch);

/*
 * Line-level update (reference kernels.py:212-247): interior line (k, j).
 * Jacobi writes dst from src (distinct buffers); GS updates src in place
 * (dst ignored).  Bounds are checked (SB_ERR_ARGUMENT).  Asynchronous.
 */
int sb_line_update(int kernel, const double* src, double* dst, int64_t ni, int64_t nj,
                   int64_t nk, int64_t k, int64_t j, double a, double b, void* stream);

/*
 * Host-buffer entry point: the whole reference `run` contract in one call.
 * host_grid: padded grid in host memory (pinned or pageable), updated in
 * place with the final field.  Copies to device `device`, sweeps, copies
 * back; synchronous.  For Jacobi a = centre weight, depth as in sb_jacobi;
 * for GS a and depth are ignored.
 */
int sb_run_host(int kernel, double* host_grid, int64_t ni, int64_t nj, int64_t nk,
                int64_t iters, double a, double b, int depth, int device);

/*
 * Batch form of sb_run_host for a stream of independent grids of one shape
 * (the reference's perf.measure runs fresh inputs back to back): entry i's
 * host->device copy overlaps entry i-1's sweeps and entry i-2's
 * device->host copy (PCIe is full duplex), so with pinned grids the batch
 * moves at about max(H2D, sweeps, D2H) per grid.  Entries are processed in
 * order; an entry may repeat the pointer of an entry at least two places
 * earlier and then starts from that entry's result (its upload waits for
 * that download); adjacent repeats -> SB_ERR_ARGUMENT.  Synchronous; every
 * grid is updated in place.  Uses three device slots (Jacobi: six grids'
 * worth of device memory), two if the third does not fit.
 */
int sb_run_host_batch(int kernel, double* const* host_grids, int count, int64_t ni, int64_t nj,
                      int64_t nk, int64_t iters, double a, double b, int depth, int device);

/*
 * Device bandwidth probe: a[i] = b[i] + s*c[i] for n doubles (device
 * pointers, 16-byte aligned), the STREAM triad of the reference's
 * perf.stream_triad (pkg/src/stencilbench/perf.py:139-211) on the GPU.
 * 24 bytes per element move.  Asynchronous on `stream`.
 */
int sb_triad(double* a, const double* b, const double* c, double s, int64_t n, void* stream);

/*
 * FP64 pipe probe: one launch of independent double-precision add chains
 * (no memory traffic) filling every SM; *ops receives the number of DP
 * operations it executes, so ops / elapsed time is the device's sustained
 * FP64 issue rate -- the secondary (compute) ceiling of the stencil kernels
 * (SURVEY.md 8(d)).  `sink` is a device buffer of >= 256 doubles (written
 * only to keep the chains alive).  Asynchronous on `stream`.
 */
int sb_fp64_probe(double* sink, int64_t iters, void* stream, int64_t* ops);

/*
 * Frees the device buffers the library keeps between calls on `device` (all
 * devices if < 0): the host-entry slots of sb_run_host / sb_run_host_batch
 * (the batch holds up to six grids' worth) and the pitched copies used for
 * odd ni.  Synchronises those devices first.  Small per-shape state (work
 * lists, counters) stays.  The next call reallocates what it needs.
 */
int sb_release_caches(int device);

/*
 * Pinned host allocation for grids (so sb_run_host copies at full PCIe
 * rate).  Returns NULL on failure.
 */
double* sb_host_alloc(int64_t count);
void sb_host_free(double* p);

/*
 * One block of `sweeps` (1..sb_max_depth()) fused Jacobi sweeps src -> dst
 * that writes only the output planes [k_out_lo, k_out_hi) (padded plane
 * indices within [1, nk]); every other plane of dst is left untouched.
 * The building block of the z-slab decomposition: a slab computes the
 * planes its neighbours need first, then its interior while those travel.
 * Values are exact wherever the input is valid `sweeps` planes beyond the
 * output range.  Asynchronous on `stream`.
 */
int sb_jacobi_planes(const double* src, double* dst, int64_t ni, int64_t nj, int64_t nk,
                     int64_t k_out_lo, int64_t k_out_hi, int sweeps, double a, double b,
                     void* stream);

/*
 * Layout of slab `slab` of the z-slab decomposition of nk interior planes
 * into `nslabs` slabs (partition_blocks semantics, sweeps/plan.py:106-120):
 * it owns global padded planes [*own_lo, *own_hi) and stores *ghost_lo
 * planes below and *ghost_hi above them (`depth` toward a neighbour slab, 1
 * -- the Dirichlet halo plane -- at the global boundary).  The slab buffer
 * is therefore a padded grid of (own_hi-own_lo + ghost_lo + ghost_hi)
 * planes holding global planes [own_lo-ghost_lo, own_hi+ghost_hi).
 * SB_ERR_PARTITION when nslabs > nk or an inner slab owns < depth planes.
 */
int sb_slab_layout(int64_t nk, int nslabs, int slab, int depth, int64_t* own_lo, int64_t* own_hi,
                   int64_t* ghost_lo, int64_t* ghost_hi);

/*
 * Multi-slab Jacobi in one process: slabs[s] / scratch[s] are device
 * buffers on devices[s] laid out per sb_slab_layout (slabs[s] filled with
 * the initial field including ghosts; scratch[s] needs no initialisation),
 * streams[s] a stream on devices[s].  Runs `iters` sweeps, `depth` per halo
 * exchange (peer copies over NVLink between GPUs, device copies between
 * slabs sharing a GPU), overlapping each exchange with the slab interiors.
 * Synchronous.  *result_in_scratch tells which buffer set holds the result
 * (owned planes exact; ghost planes are not meaningful afterwards).
 */
int sb_jacobi_slabs(int nslabs, const int* devices, double* const* slabs,
                    double* const* scratch, int64_t ni, int64_t nj, int64_t nk,
                    int64_t iters, double a, double b, int depth, void* const* streams,
                    int* result_in_scratch);

/*
 * Gauss-Seidel slab layout: slab `slab` of nslabs owns the global padded
 * planes [*own_lo, *own_hi) (partition_blocks(nk, nslabs)); its local grid
 * holds global planes own_lo-1 .. own_hi, i.e. (own_hi-own_lo) interior
 * planes between two ghost planes.  SB_ERR_PARTITION when nslabs > nk.
 */
int sb_gs_slab_layout(int64_t nk, int nslabs, int slab, int64_t* own_lo, int64_t* own_hi);

/*
 * Multi-slab Gauss-Seidel in one process (the cross-GPU z-pipeline):
 * slabs[g] is a device grid on devices[g] laid out per sb_gs_slab_layout and
 * filled with the initial global planes own_lo-1 .. own_hi; streams[g] a
 * stream on devices[g] (slabs sharing a device must share its stream).
 * Runs `iters` in-place sweeps of `kernel` (SB_KERNEL_GS_*): sweep s of slab
 * g starts once slab g-1 finished sweep s and slab g+1 sweep s-1 (ghost
 * planes copied between them), so slabs on different GPUs run as a
 * pipeline.  Owned planes end bitwise equal to sb_gs on the whole grid.
 * Synchronous.
 */
int sb_gs_slabs(int nslabs, const int* devices, double* const* slabs, int64_t ni, int64_t nj,
                int64_t nk, int64_t iters, double b, int kernel, void* const* streams);

/*
 * Multi-GPU host entry: the reference `run(plan, g)` with a threaded plan
 * spread over GPUs -- run_threaded_jacobi's k-slabs (sweeps/threaded.py:
 * 28-59, partition_blocks at :39) and run_pipeline_gs's pipelined order
 * (:62-96) with one z-slab per entry of devices[0..ndev) (an index may
 * repeat: those slabs share the GPU).  `grid` is the whole padded grid in
 * host memory or in any device's memory (UVA), updated in place with the
 * final field.  Scatters the slabs (with ghost planes), runs sb_jacobi_slabs
 * (`depth` sweeps per halo exchange, capped at the thinnest slab) or
 * sb_gs_slabs, gathers the owned planes back; slab buffers are allocated
 * for the call and freed before it returns.  Synchronous.  Bitwise equal to
 * sb_run_host.  SB_ERR_PARTITION when ndev > nk.
 */
int sb_run_multi(int kernel, double* grid, int64_t ni, int64_t nj, int64_t nk, int64_t iters,
                 double a, double b, int depth, int ndev, const int* devices);

#ifdef __cplusplus
}
#endif

#endif /* STENCIL_B200_H */
