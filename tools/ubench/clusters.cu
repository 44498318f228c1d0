// How many thread-block clusters of size 1/2/4/8 fit at once with one
// ~200 KB CTA per SM (decides whether a cluster-based stencil loses SMs).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dummy(int* p) { extern __shared__ int s[]; if (p) p[0] = s[threadIdx.x]; }
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int cs : {1, 2, 4, 8, 16}) {
        for (int smem : {100 * 1024, 200 * 1024}) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(cs * 64); cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = smem;
            cudaLaunchAttribute at; at.id = cudaLaunchAttributeClusterDimension;
            at.val.clusterDim.x = cs; at.val.clusterDim.y = 1; at.val.clusterDim.z = 1;
            cfg.attrs = &at; cfg.numAttrs = 1;
            int n = -1;
            cudaError_t e = cudaOccupancyMaxActiveClusters(&n, dummy, &cfg);
            printf("cluster %2d smem %3d KB: max active clusters %d -> %d CTAs of %d SMs (%s)\n", cs,
                   smem / 1024, n, n * cs, sms, cudaGetErrorString(e));
        }
    }
}
