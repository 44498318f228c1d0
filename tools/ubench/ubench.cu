// Microbenchmarks of B200 primitives relevant to the stencil kernels.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dadd_chain(double* out, double x, int n, long long* cyc) {
    double a = x + threadIdx.x, b = 1e-300;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        a = __dadd_rn(a, b); a = __dadd_rn(a, b); a = __dadd_rn(a, b); a = __dadd_rn(a, b);
    }
    long long t1 = clock64();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void dmul_chain(double* out, double x, int n, long long* cyc) {
    double a = x + threadIdx.x, b = 1.0000001;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        a = __dmul_rn(a, b); a = __dmul_rn(a, b); a = __dmul_rn(a, b); a = __dmul_rn(a, b);
    }
    long long t1 = clock64();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void bar_loop(int n, long long* cyc) {
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) asm volatile("bar.sync 1, %0;" :: "r"(blockDim.x));
    long long t1 = clock64();
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void lds_chain(int n, long long* cyc, int* out) {
    __shared__ int s[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (i + 1) & 1023;
    __syncthreads();
    int p = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) p = s[p];
    long long t1 = clock64();
    out[threadIdx.x] = p;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
// synthetic GS step: 5 LDS + 6-op DP chain + STS + named barrier; lanes
// skewed by one column like the real tile (line L at column st - L)
__global__ void gs_step(int n, long long* cyc, double* out) {
    __shared__ double s[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = 1.0 / (i + 1);
    __syncthreads();
    const int L = threadIdx.x;
    const int Ls = (L + 255) & 255, Ln = (L + 1) & 255, Ld = (L + 240) & 255, Lu = (L + 16) & 255;
    double w = 0.5, b = 1.0 / 6.0;
    long long t0 = clock64();
    for (int st = 0; st < n; ++st) {
        const int c = (st - L) & 15;
        double e = s[L * 16 + ((c + 1) & 15)];
        double sv = s[Ls * 16 + c], nv = s[Ln * 16 + c];
        double dv = s[Ld * 16 + c], uv = s[Lu * 16 + c];
        double acc = __dadd_rn(w, e);
        acc = __dadd_rn(acc, sv); acc = __dadd_rn(acc, nv); acc = __dadd_rn(acc, dv); acc = __dadd_rn(acc, uv);
        double x = __dmul_rn(b, acc);
        s[L * 16 + c] = x;
        w = x;
        asm volatile("bar.sync 1, %0;" :: "r"(blockDim.x));
    }
    long long t1 = clock64();
    out[threadIdx.x] = w;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
    double* out; long long* cyc; int* iout;
    cudaMalloc(&out, 1 << 16); cudaMalloc(&cyc, 8); cudaMalloc(&iout, 1 << 16);
    long long h;
    const int n = 4096;
    dadd_chain<<<1, 32>>>(out, 1.0, n, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("DADD dependent latency: %.2f cycles\n", (double)h / (4.0 * n));
    dmul_chain<<<1, 32>>>(out, 1.0, n, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("DMUL dependent latency: %.2f cycles\n", (double)h / (4.0 * n));
    for (int t : {32, 64, 128, 256, 512}) {
        bar_loop<<<1, t>>>(n, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("bar.sync (%d threads): %.2f cycles\n", t, (double)h / n);
    }
    lds_chain<<<1, 32>>>(n, cyc, iout); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("LDS dependent latency: %.2f cycles\n", (double)h / n);
    for (int t : {32, 128, 256}) {
        gs_step<<<1, t>>>(n, cyc, out); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("synthetic GS step (%d threads, 1 CTA): %.2f cycles\n", t, (double)h / n);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
