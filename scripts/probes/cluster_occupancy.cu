// How many clusters of size 1/2/4/8 fit at once with one 384-thread CTA per SM
// using ~230 KB of dynamic shared memory (the GEMM kernel's footprint).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dummy(int *p) { if (p) p[threadIdx.x] = 0; }
int main() {
    cudaFuncSetAttribute(dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, 230656);
    cudaFuncSetAttribute(dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int cs : {1, 2, 4, 8, 16}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cs * 64); cfg.blockDim = dim3(384); cfg.dynamicSmemBytes = 230656;
        cudaLaunchAttribute a; a.id = cudaLaunchAttributeClusterDimension;
        a.val.clusterDim.x = cs; a.val.clusterDim.y = 1; a.val.clusterDim.z = 1;
        cfg.attrs = &a; cfg.numAttrs = 1;
        int n = -1; cudaError_t e = cudaOccupancyMaxActiveClusters(&n, dummy, &cfg);
        printf("cluster %2d: max active clusters %3d -> %3d SMs of %d (%s)\n", cs, n, n * cs, sms, cudaGetErrorString(e));
    }
    return 0;
}
