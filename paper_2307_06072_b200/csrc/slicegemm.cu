// slicegemm.cu -- the triangle of slice products of Algorithm 2 on the
// sm_100a INT8 tensor cores.
//
// For every work unit (job, output tile, anti-diagonal r, k-block chunk [g0, g1)) it
// computes, exactly in INT32,
//     D = sum_{g in [g0,g1)}  A_{pa, p}[tile rows, kb] . B_{pb, r-p}[tile cols, kb]^T
// where g enumerates (pair, p = 1..r-1, kb) of the job's concatenated K' = npairs (r-1) k,
// i.e. one chunk of  D_r = sum_{alpha+beta=r} A_alpha B_beta  (the anti-diagonal form of
// the triangle beta <= d - alpha + 1), and stores D to partial plane `slot`.
//
// Kernel structure (one CTA per SM, persistent over a host-balanced unit list):
//   warp 0 lane 0 : TMA producer, STAGES-deep ring of (A 128x128 B, B BNx128 B) int8 tiles
//   warp 1        : TMEM allocator; lane 0 issues tcgen05.mma.cta_group::1.kind::i8
//                   (M=128, N=BN, K=32; 4 per 128-byte k-block) into a double-buffered
//                   TMEM accumulator (2 x BN columns)
//   warps 4..7    : epilogue, tcgen05.ld 32x32b -> registers -> int32 partial plane
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include "common.cuh"
#include "kernels.h"

namespace mpc {

constexpr int kBM = 128;

template <int BN, int STAGES>
struct TcCfg {
    static constexpr int A_BYTES = kBM * kBK;
    static constexpr int B_BYTES = BN * kBK;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int TMEM_COLS = 2 * BN;
    static constexpr size_t SMEM = 1024 /*align slack*/ + (size_t)STAGES * STAGE_BYTES + 256 /*barriers*/;
};

template <int BN, int STAGES>
__global__ void __launch_bounds__(256, 1)
slicegemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ GemmParams P)
{
    using Cfg = TcCfg<BN, STAGES>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *sA = smem;
    uint8_t *sB = smem + STAGES * Cfg::A_BYTES;
    uint64_t *full = reinterpret_cast<uint64_t *>(sB + STAGES * Cfg::B_BYTES);
    uint64_t *empty = full + STAGES;
    uint64_t *tfull = empty + STAGES;
    uint64_t *tempty = tfull + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0 && lane == 0) {
        for (int i = 0; i < STAGES; i++) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
        for (int i = 0; i < 2; i++) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], 128); }
        fence_barrier_init();
        tma_prefetch(&tmA);
        tma_prefetch(&tmB);
    }
    if (warp == 1) tmem_alloc<Cfg::TMEM_COLS>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const int ubeg = P.cta_begin[blockIdx.x], uend = P.cta_begin[blockIdx.x + 1];
    const int s = P.s, KB = P.KB;

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- TMA producer
            int stage = 0; uint32_t phase = 0;
            for (int u = ubeg; u < uend; u++) {
                const WorkUnit w = P.units[u];
                const JobDesc &J = P.jobs[w.job];
                const int per_pair = (w.r - 1) * KB;
                for (int g = w.g0; g < w.g1; g++) {
                    const int pair = g / per_pair;
                    const int rem = g - pair * per_pair;
                    const int p0 = rem / KB;              // alpha - 1
                    const int kb = rem - p0 * KB;
                    const int planeA = J.pa[pair] * s + p0;
                    const int planeB = J.pb[pair] * s + (w.r - 2 - p0);   // beta - 1, beta = r - alpha
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_arrive_expect_tx(&full[stage], Cfg::STAGE_BYTES);
                    tma_load_3d(sA + stage * Cfg::A_BYTES, &tmA, &full[stage], kb * kBK, w.tm * kBM, planeA);
                    tma_load_3d(sB + stage * Cfg::B_BYTES, &tmB, &full[stage], kb * kBK, w.tn * BN, planeB);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (lane == 0) {
            // ---------------- MMA issuer
            constexpr uint32_t idesc = make_idesc_i8(kBM, BN);
            int stage = 0; uint32_t phase = 0;
            int buf = 0; uint32_t tphase = 0;
            for (int u = ubeg; u < uend; u++) {
                const WorkUnit w = P.units[u];
                mbar_wait(&tempty[buf], tphase ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + (uint32_t)(buf * BN);
                for (int g = w.g0; g < w.g1; g++) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(sA + stage * Cfg::A_BYTES);
                    const uint32_t b0 = smem_u32(sB + stage * Cfg::B_BYTES);
#pragma unroll
                    for (int kk = 0; kk < kBK / 32; kk++) {
                        mma_i8(d_tmem, make_sw128_desc(a0 + kk * 32), make_sw128_desc(b0 + kk * 32), idesc,
                               (g > w.g0 || kk > 0) ? 1u : 0u);
                    }
                    mma_commit(&empty[stage]);                // frees the smem slot when done
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
                mma_commit(&tfull[buf]);                      // accumulator ready
                buf ^= 1; if (buf == 0) tphase ^= 1;
            }
        }
        __syncwarp();
    } else if (warp >= 4) {
        // ---------------- epilogue: TMEM -> registers -> int32 partial plane
        const int q = warp & 3;                               // TMEM lane quarter of this warp
        int buf = 0; uint32_t tphase = 0;
        for (int u = ubeg; u < uend; u++) {
            const WorkUnit w = P.units[u];
            mbar_wait(&tfull[buf], tphase);
            tc_fence_after();
            const int row = w.tm * kBM + q * 32 + lane;
            int32_t *out = P.partials + (int64_t)w.slot * P.plane + (int64_t)row * P.ldD;
#pragma unroll 1
            for (int c = 0; c < BN / 32; c++) {
                uint32_t v[32];
                tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * BN + c * 32), v);
                tmem_ld_wait();
                const int col0 = w.tn * BN + c * 32;
                if (row < P.m) {
#pragma unroll
                    for (int g4 = 0; g4 < 8; g4++) {
                        if (col0 + 4 * g4 < P.ldD) {
                            int4 val = make_int4((int)v[4 * g4], (int)v[4 * g4 + 1], (int)v[4 * g4 + 2], (int)v[4 * g4 + 3]);
                            *reinterpret_cast<int4 *>(out + col0 + 4 * g4) = val;
                        }
                    }
                }
            }
            tc_fence_before();
            mbar_arrive(&tempty[buf]);
            buf ^= 1; if (buf == 0) tphase ^= 1;
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) tmem_dealloc<Cfg::TMEM_COLS>(tmem_base);
}

// ------------------------------------------------------------------ SIMT cross-check kernel
// Same work list and output, computed with dp4a on CUDA cores (used by the tests to check
// the tensor-core kernel bitwise; selected with MPCGEMM_SLICEGEMM=simt).  One CTA per
// (unit, 32x32 subtile), one thread per output element.
__global__ void __launch_bounds__(256)
slicegemm_simt_kernel(const int8_t *__restrict__ digA, const int8_t *__restrict__ digB,
                      int64_t rowsA, int64_t rowsB, int64_t kp, const WorkUnit *units, int BN,
                      const GemmParams P)
{
    __shared__ int32_t sa[32][kBK / 4 + 1];
    __shared__ int32_t sb[32][kBK / 4 + 1];
    const WorkUnit w = units[blockIdx.x];
    const JobDesc &J = P.jobs[w.job];
    const int sub = blockIdx.y;                   // 32x32 subtile index within 128 x BN
    const int sub_m = sub % (kBM / 32), sub_n = sub / (kBM / 32);
    const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;   // 32 x 8
    const int64_t row0 = (int64_t)w.tm * kBM + sub_m * 32;
    const int64_t col0 = (int64_t)w.tn * BN + sub_n * 32;
    int32_t acc[4] = {0, 0, 0, 0};
    const int per_pair = (w.r - 1) * P.KB;
    for (int g = w.g0; g < w.g1; g++) {
        const int pair = g / per_pair;
        const int rem = g - pair * per_pair;
        const int p0 = rem / P.KB;
        const int kb = rem - p0 * P.KB;
        const int8_t *pa = digA + ((int64_t)(J.pa[pair] * P.s + p0) * rowsA) * kp;
        const int8_t *pb = digB + ((int64_t)(J.pb[pair] * P.s + (w.r - 2 - p0)) * rowsB) * kp;
        __syncthreads();
        for (int t = threadIdx.x; t < 32 * (kBK / 4); t += 256) {
            int rr = t / (kBK / 4), cc = t % (kBK / 4);
            int64_t kk = (int64_t)kb * kBK + cc * 4;
            int32_t va = 0, vb = 0;
            if (row0 + rr < rowsA && kk < kp) va = *reinterpret_cast<const int32_t *>(pa + (row0 + rr) * kp + kk);
            if (col0 + rr < rowsB && kk < kp) vb = *reinterpret_cast<const int32_t *>(pb + (col0 + rr) * kp + kk);
            sa[rr][cc] = va; sb[rr][cc] = vb;
        }
        __syncthreads();
        for (int e = 0; e < 4; e++) {
            const int r_ = ty * 4 + e;
#pragma unroll 8
            for (int cc = 0; cc < kBK / 4; cc++) acc[e] = __dp4a(sa[r_][cc], sb[tx][cc], acc[e]);
        }
    }
    for (int e = 0; e < 4; e++) {
        const int64_t row = row0 + ty * 4 + e, col = col0 + tx;
        if (row < P.m && col < P.ldD) P.partials[(int64_t)w.slot * P.plane + row * P.ldD + col] = acc[e];
    }
}

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void *p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// 3-D map over digit planes int8 [planes][rows][kp] with box {128, box_rows, 1}, 128B swizzle
static int make_plane_map(CUtensorMap *map, const int8_t *base, int64_t planes, int64_t rows, int64_t kp, int box_rows) {
    auto enc = get_encode();
    if (!enc) return -1;
    cuuint64_t dims[3] = {(cuuint64_t)kp, (cuuint64_t)rows, (cuuint64_t)planes};
    cuuint64_t strides[2] = {(cuuint64_t)kp, (cuuint64_t)(kp * rows)};
    cuuint32_t box[3] = {(cuuint32_t)kBK, (cuuint32_t)box_rows, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t *>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : -2;
}

template <int BN, int STAGES>
static cudaError_t launch_tc(const SliceGemmLaunch &L, cudaStream_t st) {
    using Cfg = TcCfg<BN, STAGES>;
    CUtensorMap ta, tb;
    if (make_plane_map(&ta, L.digA, (int64_t)L.P.partsA * L.P.s, L.rowsA, L.kp, kBM)) return cudaErrorInvalidValue;
    if (make_plane_map(&tb, L.digB, (int64_t)L.P.partsB * L.P.s, L.rowsB, L.kp, BN)) return cudaErrorInvalidValue;
    auto kern = slicegemm_tc_kernel<BN, STAGES>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM);
    if (e != cudaSuccess) return e;
    kern<<<L.grid, 256, Cfg::SMEM, st>>>(ta, tb, L.P);
    return cudaGetLastError();
}

cudaError_t slicegemm_launch(const SliceGemmLaunch &L, cudaStream_t st) {
    if (L.grid <= 0) return cudaSuccess;
    if (L.simt) {
        dim3 grid(L.nunits, (kBM / 32) * (L.BN / 32));
        slicegemm_simt_kernel<<<grid, 256, 0, st>>>(L.digA, L.digB, L.rowsA, L.rowsB, L.kp, L.units_flat, L.BN, L.P);
        return cudaGetLastError();
    }
    if (L.BN == 256) return launch_tc<256, 4>(L, st);
    if (L.BN == 128) return launch_tc<128, 6>(L, st);
    return cudaErrorInvalidValue;
}

}  // namespace mpc
