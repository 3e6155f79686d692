// mma_shape.cu -- (variant of mma_power.cu, N = NN) microbenchmark (not part of the library): back-to-back tcgen05.mma kind::i8
// (M=128, N=256, K=32) on operands resident in shared memory, one CTA per SM, ~3 s.  Reports
// INT8 TOP/s and the effective SM clock (clock64 / globaltimer), i.e. the power-capped ceiling
// of the tensor pipe without any TMA / L2 / HBM traffic.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2307_06072_b200/csrc mma_power.cu -o mma_power
#include <cstdio>
#include <cstdlib>
#include "common.cuh"
#ifndef NSTAGE
#define NSTAGE 4
#endif
#ifndef NN
#define NN 256
#endif

using namespace mpc;

__global__ void __launch_bounds__(128, 1) mma_loop(long long iters, unsigned long long *cycles, unsigned long long *nanos) {
    extern __shared__ __align__(1024) uint8_t sm[];
    constexpr int NS = NSTAGE;                       // rotating operand stages (input toggling)
    uint8_t *sA = sm, *sB = sm + NS * 16384;  // B stage NN*128 bytes
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + NS * (16384 + NN * 128));
    uint32_t *slot = reinterpret_cast<uint32_t *>(bar + 1);
    uint32_t x = 2463534242u ^ (blockIdx.x * 7919u + threadIdx.x * 104729u);
    for (int i = threadIdx.x; i < NS * (16384 + NN * 128) / 4; i += blockDim.x) {
        x ^= x << 13; x ^= x >> 17; x ^= x << 5;     // xorshift: random digits
        reinterpret_cast<uint32_t *>(sm)[i] = x;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x == 0) { mbar_init(bar, 1); fence_barrier_init(); }
    if (threadIdx.x < 32) tmem_alloc<512>(slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tm = *slot;
    unsigned long long c0 = clock64(), t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    if (threadIdx.x == 0) {
        const uint32_t idesc = make_idesc_i8(128, NN);
        uint32_t ph = 0;
        for (long long it = 0; it < iters; it++) {
            const uint32_t a0 = smem_u32(sA + (it % NS) * 16384), b0 = smem_u32(sB + (it % NS) * (NN * 128));
#pragma unroll
            for (int kk = 0; kk < 4; kk++)
                mma_i8(tm + (uint32_t)((it & 1) * NN), make_sw128_desc(a0 + kk * 32), make_sw128_desc(b0 + kk * 32), idesc, 1u);
            if ((it & 63) == 63) { mma_commit(bar); mbar_wait(bar, ph); ph ^= 1; }
        }
        mma_commit(bar); mbar_wait(bar, ph);
    }
    __syncthreads();
    unsigned long long c1 = clock64(), t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (threadIdx.x == 0) { cycles[blockIdx.x] = c1 - c0; nanos[blockIdx.x] = t1 - t0; }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x < 32) tmem_dealloc<512>(tm);
}

int main(int argc, char **argv) {
    long long iters = argc > 1 ? atoll(argv[1]) : 60000;
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long *cyc, *ns;
    cudaMalloc(&cyc, 8 * nsm); cudaMalloc(&ns, 8 * nsm);
    size_t smem = NSTAGE * (16384 + NN * 128) + 64;
    cudaFuncSetAttribute(mma_loop, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    mma_loop<<<nsm, 128, smem>>>(iters / 10, cyc, ns);           // warm-up
    cudaDeviceSynchronize();
    mma_loop<<<nsm, 128, smem>>>(iters, cyc, ns);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    unsigned long long hc[1024], hn[1024];
    cudaMemcpy(hc, cyc, 8 * nsm, cudaMemcpyDeviceToHost);
    cudaMemcpy(hn, ns, 8 * nsm, cudaMemcpyDeviceToHost);
    double maxns = 0, sumclk = 0;
    for (int i = 0; i < nsm; i++) { if (hn[i] > maxns) maxns = (double)hn[i]; sumclk += (double)hc[i] / (double)hn[i]; }
    const double ops = 2.0 * 128 * NN * 128.0 * (double)iters * nsm;   // 4 x K=32 per iteration
    printf("{\"int8_tops\": %.1f, \"seconds\": %.3f, \"avg_sm_ghz\": %.3f, \"cycles_per_mma\": %.2f}\n", ops / (maxns * 1e-9) / 1e12,
           maxns * 1e-9, sumclk / nsm, (double)hc[0] / (4.0 * (double)iters));
    return 0;
}
