// probe: 4-D TMA store of [parts][8 planes][128 k] staged bytes into digit planes (split TS path)
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <vector>
#include "../paper_2307_06072_b200/csrc/common.cuh"
using namespace mpc;
__global__ void probe(const __grid_constant__ CUtensorMap om, int s, int c2) {
    extern __shared__ __align__(1024) uint8_t sm[];
    for (int i = threadIdx.x; i < 3 * 8 * 128; i += blockDim.x) sm[i] = (uint8_t)(i % 251 + 1);
    fence_proxy_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) { tma_store_4d(&om, sm, 0, 1, c2, 0); bulk_commit(); bulk_wait<0>(); }
}
int main() {
    const int kp = 64, lines = 64, s = 17, parts = 3;
    int8_t *dig; cudaMalloc(&dig, (size_t)kp * lines * s * parts); cudaMemset(dig, 0, (size_t)kp * lines * s * parts);
    cudaDriverEntryPointQueryResult q; void *p = nullptr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    alignas(64) CUtensorMap m;
    cuuint64_t dims[4] = {(cuuint64_t)kp, (cuuint64_t)lines, (cuuint64_t)s, (cuuint64_t)parts};
    cuuint64_t strides[3] = {(cuuint64_t)kp, (cuuint64_t)(kp * lines), (cuuint64_t)(kp * lines * s)};
    cuuint32_t box[4] = {128, 1, 8, (cuuint32_t)parts};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, dig, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d\n", (int)r);
    for (int c2 : {s - 8, 0}) {
        cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
        probe<<<1, 128, 8192>>>(m, s, c2);
        cudaError_t e = cudaDeviceSynchronize();
        printf("c2=%d: %s\n", c2, cudaGetErrorString(e));
        if (e != cudaSuccess) return 1;
    }
    std::vector<int8_t> h((size_t)kp * lines * s * parts);
    cudaMemcpy(h.data(), dig, h.size(), cudaMemcpyDeviceToHost);
    // plane s-1 of part 0, line 1, kk 0..3 should be staging row 7 bytes
    printf("part0 plane%d line1: %d %d  (expect %d %d)\n", s - 1, h[((0 * s + s - 1) * lines + 1) * kp + 0],
           h[((0 * s + s - 1) * lines + 1) * kp + 1], (int8_t)((7 * 128) % 251 + 1), (int8_t)((7 * 128 + 1) % 251 + 1));
    return 0;
}
