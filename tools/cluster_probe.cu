// max co-resident clusters of 2 / 4 / 8 CTAs (one 216 KB-smem CTA per SM), as the slice GEMM
// would launch them -- is a 4-CTA cluster (two CTA pairs sharing B by multicast) worth the SMs?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dummy(int *p) { extern __shared__ int s[]; if (p) p[0] = s[0]; }
int main() {
    const int smem = 216 * 1024 + 576;
    cudaFuncSetAttribute(dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int cs : {1, 2, 4, 8, 16}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cs * 64); cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        int n = -1;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&n, dummy, &cfg);
        printf("cluster %2d: max active clusters %d (%d SMs) %s\n", cs, n, n * cs, cudaGetErrorString(e));
    }
}
