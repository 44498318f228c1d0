// sb_internal.h -- declarations shared by the library's translation units.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdlib>
#include <vector>

namespace sb {

struct JacPeers;  // jacobi_tb.cuh

// Tuning knobs (SB_KBLK, SB_LIST*, SB_GS_WINDOW, SB_GSCFG, SB_JCFG) are read
// from the environment only in experiment builds (-DSB_EXPERIMENTS, tools/);
// the product library always runs its measured defaults.
inline const char* tune_env(const char* name) {
#ifdef SB_EXPERIMENTS
    return getenv(name);
#else
    (void)name;
    return nullptr;
#endif
}

int fail(int code, const char* fmt, ...);

// Restores the caller's current device when an entry point that switches
// devices returns (any path).
struct DeviceGuard {
    int dev = -1;
    DeviceGuard() {
        if (cudaGetDevice(&dev) != cudaSuccess) {
            cudaGetLastError();
            dev = -1;
        }
    }
    ~DeviceGuard() {
        if (dev >= 0) cudaSetDevice(dev);
    }
    DeviceGuard(const DeviceGuard&) = delete;
    DeviceGuard& operator=(const DeviceGuard&) = delete;
};

// Resident CTAs per SM of `kern` on the current device, with its dynamic
// shared-memory opt-in made first.  The opt-in is a property of each
// device's context, so it is made once per (kernel, device) -- not once per
// process (sb_api.cu).
int ctas_per_sm(const void* kern, int threads, size_t smem, int* out);
int cuda_fail(cudaError_t e, const char* what);
void clear_error();
const char* last_error();

int check_dims(int64_t ni, int64_t nj, int64_t nk);
int make_grid_map3p(CUtensorMap* m, const double* base, int64_t nip, int64_t njp, int64_t nkp,
                    int bw, int bh, int bd, int64_t pitch);
int get_counters(int** counters, int* sms);
bool tma_ok(const void* p, int64_t ni);
int halo_copy(const double* src, double* dst, int ni, int nj, int nk, cudaStream_t st);
int jacobi_block(const double* src, double* dst, int ni, int nj, int nk, int kfirst, int klast,
                 int T, double a, double b, cudaStream_t st, const JacPeers* peers = nullptr);
int jacobi_run(double* a_buf, double* b_buf, int ni, int nj, int nk, int64_t iters, double a,
               double b, int depth, cudaStream_t st, int* in_b);
int jacobi_generic_sweep(const double* src, double* dst, int ni, int nj, int nk, double a, double b,
                         cudaStream_t st);
int gs_run(double* grid, int ni, int nj, int nk, int64_t iters, double b, int kernel,
           cudaStream_t st);
int gs_slabs_fused(int nslabs, const int* devices, double* const* grids, const int64_t* nks, int ni,
                   int nj, int64_t iters, double b, int kernel, void* const* streams);
int gs_check_error(cudaStream_t st);
bool peer_reachable(int a, int b);  // kernels on a may store into b's memory

// work schedules of the temporally blocked Jacobi launch (sched.cu)
int64_t schedule_span(int T, int tiles, int nkout, int grid, int kb);
int pick_kblock(int T, int tiles, int nkout, int grid);
std::vector<int4> build_item_list(int T, int tiles_i, int tiles_j, const std::vector<char>& border,
                                  int kfirst, int klast, int grid, int kb);
int item_list(int T, int tiles_i, int tiles_j, const std::vector<char>& border, int kfirst,
              int klast, int grid, int kb, bool regular_only, const int4** out, int* count);

// free the per-device buffers kept between calls; true if there were any
bool gs_release(int dev);
bool jacobi_release(int dev);
bool gs_holds(int dev);
bool jacobi_holds(int dev);

}  // namespace sb
