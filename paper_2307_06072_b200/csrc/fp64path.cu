// fp64path.cu -- NEXT-1: the same Ozaki method with the paper's own slice
// carrier, binary64 slices of b = 53 - ceil((53 + ceil(log2 k)) / 2) bits (Algorithm 2's tau,
// PAPER.md:161) multiplied on the FP64 tensor cores (DMMA, mma.sync.m16n8k8.f64; tcgen05 has no
// f64 kind).  The result is bit-identical to oracle/mpref.c orc_cgemm_ozaki_bits(b) for the same
// number of divisions d:
//   split  : X = sign floor(|x| 2^(W-e)), W = b d - 3; its d balanced radix-2^b digits as doubles
//   gemm   : D_r = sum_{alpha+beta=r} A_alpha B_beta; every pair product is an integer of
//            magnitude <= k 2^(2b-2) <= 2^51, exact in binary64 (the point of the paper's b); up
//            to 4 pair products are summed in fp64 (<= 2^53, still exact), then flushed to int64
//   fold   : Eq. 5 / Eq. 6 combination, carry chain in radix 2^b, one RNE to prec
#include <cstdint>
#include "common.cuh"
#include "kernels.h"

namespace mpc {

// ------------------------------------------------------------------ split into binary64 digits
struct BitStream {          // b-bit chunks of floor(N 2^-pos), from the least significant one
    const uint64_t *N;
    int L;
    int64_t pos;
    MPC_DEV uint64_t limb(int64_t i) const { return (i >= 0 && i < L) ? __ldg(N + i) : 0ull; }
    MPC_DEV uint32_t next(int b) {
        const int64_t li = pos >= 0 ? (pos >> 6) : -((-pos + 63) >> 6);
        const int bo = (int)(pos - (li << 6));
        const uint64_t lo = limb(li), hi = limb(li + 1);
        const uint64_t v = bo ? ((lo >> bo) | (hi << (64 - bo))) : lo;
        pos += b;
        return (uint32_t)(v & ((1ull << b) - 1));
    }
};

__global__ void __launch_bounds__(128)
split_f64_kernel(DMat re, DMat im, int side, int64_t lines, int64_t k, int64_t kp, int L,
                 const int64_t *__restrict__ eline, int s, int b, int nparts, double *__restrict__ dig)
{
    const int64_t kk = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (kk >= kp) return;
    const int64_t plane = lines * kp;
    const uint32_t mask = (1u << b) - 1, half = 1u << (b - 1);
    for (int64_t line = blockIdx.y; line < lines; line += gridDim.y) {
        double *out = dig + line * kp + kk;
        BitStream bs[2];
        uint32_t neg[2], nc[2] = {1, 1};
        if (kk < k) {
            const int64_t e = eline[line];
            const int64_t W = (int64_t)b * s - 3;
            for (int p = 0; p < 2; p++) {
                const DMat &M = p ? im : re;
                const int64_t idx = side == 0 ? line * M.ld + kk : kk * M.ld + line;
                const uint64_t *N = M.limbs + idx * L;
                const bool zero = __ldg(N + L - 1) == 0;
                bs[p] = BitStream{N, zero ? 0 : L, 64 * (int64_t)L - W + e - __ldg(M.exp + idx)};
                neg[p] = zero ? 0u : (uint32_t)__ldg(M.sign + idx);
            }
        } else {
            for (int p = 0; p < 2; p++) { bs[p] = BitStream{nullptr, 0, 0}; neg[p] = 0; }
        }
        uint32_t csum = 0, rc[3] = {0, 0, 0};
        for (int t = 0; t < s; t++) {
            uint32_t y[3];
            for (int p = 0; p < 2; p++) {
                uint32_t c = bs[p].next(b);
                if (neg[p]) { const uint32_t v = (~c & mask) + nc[p]; nc[p] = v >> b; c = v & mask; }
                y[p] = c;
            }
            { const uint32_t v = y[0] + y[1] + csum; csum = v >> b; y[2] = v & mask; }
            const int64_t a = s - 1 - t;
            for (int p = 0; p < nparts; p++) {
                const uint32_t v = y[p] + rc[p];
                const int64_t d = v >= half ? (int64_t)v - (int64_t)(1u << b) : (int64_t)v;
                rc[p] = v >= half;
                out[((int64_t)p * s + a) * plane] = (double)d;
            }
        }
    }
}

cudaError_t split_f64_launch(DMat re, DMat im, int side, int64_t lines, int64_t k, int64_t kp, int L,
                             const int64_t *eline, int s, int b, int nparts, double *dig, cudaStream_t st)
{
    if (lines == 0 || kp == 0) return cudaSuccess;
    dim3 grid((unsigned)((kp + 127) / 128), (unsigned)(lines < 65535 ? lines : 65535));
    split_f64_kernel<<<grid, 128, 0, st>>>(re, im, side, lines, k, kp, L, eline, s, b, nparts, dig);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ DMMA triangle GEMM
// unit = (job, 64x64 tile, diagonal r); 4 warps, each a 32x32 sub-tile of m16n8k8 fragments.
constexpr int kDT = 64, kDK = 16, kDLd = 18;          // tile, k-step, padded smem row (doubles)

MPC_DEV void dmma_16x8x8(double (&d)[4], const double (&a)[4], const double (&b)[2]) {
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
                 : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}
MPC_DEV void cp_async16(void *dst, const void *src, bool valid) {
    const int n = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(n) : "memory");
}

__global__ void __launch_bounds__(128)
dmma_slicegemm_kernel(const double *__restrict__ digA, const double *__restrict__ digB, int64_t m, int64_t n,
                      int64_t kp, int s, const int4 *__restrict__ units, const JobDesc *__restrict__ jobs,
                      int64_t *__restrict__ partials, int64_t plane, int njobs)
{
    __shared__ __align__(16) double sA[2][kDT][kDLd];
    __shared__ __align__(16) double sB[2][kDT][kDLd];
    const int4 u = units[blockIdx.x];                  // {job, tm, tn, r}
    const JobDesc J = jobs[u.x];
    const int r = u.w;
    const int64_t row0 = (int64_t)u.y * kDT, col0 = (int64_t)u.z * kDT;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
    double acc[2][4][4];
    int64_t tot[2][4][4];
    for (int i = 0; i < 2; i++) for (int j = 0; j < 4; j++) for (int v = 0; v < 4; v++) { acc[i][j][v] = 0; tot[i][j][v] = 0; }
    const int nk = (int)(kp / kDK);
    const int npairs_total = J.npairs * (r - 1);
    int since_flush = 0;
    for (int q = 0; q < npairs_total; q++) {
        const int pr = q / (r - 1), p0 = q % (r - 1);         // alpha - 1 = p0, beta - 1 = r - 2 - p0
        const double *pa = digA + ((int64_t)(J.pa[pr] * s + p0) * m) * kp;
        const double *pb = digB + ((int64_t)(J.pb[pr] * s + (r - 2 - p0)) * n) * kp;
        auto load = [&](int buf, int kb) {
            for (int c = tid; c < kDT * kDK / 2; c += 128) {   // 16 B = 2 doubles per copy
                const int rr = c / (kDK / 2), cc = (c % (kDK / 2)) * 2;
                const int64_t ga = row0 + rr, gb = col0 + rr, gk = (int64_t)kb * kDK + cc;
                cp_async16(&sA[buf][rr][cc], pa + (ga < m ? ga : 0) * kp + gk, ga < m);
                cp_async16(&sB[buf][rr][cc], pb + (gb < n ? gb : 0) * kp + gk, gb < n);
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        };
        load(0, 0);
        for (int kb = 0; kb < nk; kb++) {
            const int buf = kb & 1;
            if (kb + 1 < nk) { load(buf ^ 1, kb + 1); asm volatile("cp.async.wait_group 1;" ::: "memory"); }
            else asm volatile("cp.async.wait_group 0;" ::: "memory");
            __syncthreads();
#pragma unroll
            for (int k8 = 0; k8 < kDK; k8 += 8) {
                double af[2][4], bf[4][2];
#pragma unroll
                for (int i = 0; i < 2; i++) {
                    const int rr = wm + i * 16 + (lane >> 2), kc = k8 + (lane & 3);
                    af[i][0] = sA[buf][rr][kc];     af[i][1] = sA[buf][rr + 8][kc];
                    af[i][2] = sA[buf][rr][kc + 4]; af[i][3] = sA[buf][rr + 8][kc + 4];
                }
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const int cc = wn + j * 8 + (lane >> 2), kc = k8 + (lane & 3);
                    bf[j][0] = sB[buf][cc][kc]; bf[j][1] = sB[buf][cc][kc + 4];
                }
#pragma unroll
                for (int i = 0; i < 2; i++)
#pragma unroll
                    for (int j = 0; j < 4; j++) dmma_16x8x8(acc[i][j], af[i], bf[j]);
            }
            __syncthreads();
        }
        if (++since_flush == 4 || q == npairs_total - 1) {  // <= 4 products: |sum| <= 2^53, exact
            for (int i = 0; i < 2; i++) for (int j = 0; j < 4; j++) for (int v = 0; v < 4; v++) {
                tot[i][j][v] += (int64_t)__double2ll_rn(acc[i][j][v]);
                acc[i][j][v] = 0;
            }
            since_flush = 0;
        }
    }
    // D_r of this job -> partial plane (job, r): slot = job * (s + 2) + r
    int64_t *out = partials + (int64_t)(u.x * (s + 2) + r) * plane;
    for (int i = 0; i < 2; i++)
        for (int j = 0; j < 4; j++)
            for (int v = 0; v < 4; v++) {
                const int64_t rr = row0 + wm + i * 16 + (lane >> 2) + (v >> 1) * 8;
                const int64_t cc = col0 + wn + j * 8 + 2 * (lane & 3) + (v & 1);
                if (rr < m && cc < n) out[rr * n + cc] = tot[i][j][v];
            }
}

cudaError_t dmma_slicegemm_launch(const double *digA, const double *digB, int64_t m, int64_t n, int64_t kp, int s,
                                  const int4 *units, int nunits, const JobDesc *jobs, int njobs, int64_t *partials,
                                  cudaStream_t st)
{
    if (nunits == 0) return cudaSuccess;
    dmma_slicegemm_kernel<<<nunits, 128, 0, st>>>(digA, digB, m, n, kp, s, units, jobs, partials, m * n, njobs);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ fold in radix 2^b + RNE
MPC_DEV void round_store_local(const uint64_t *mag, int n, int64_t e_lsb, bool neg, int prec, int L,
                               uint8_t *sign_out, int64_t *exp_out, uint64_t *limbs_out)
{
    int bl = 0;
    for (int l = n - 1; l >= 0; l--) if (mag[l]) { bl = 64 * l + 64 - __clzll((long long)mag[l]); break; }
    if (bl == 0) { *sign_out = 0; *exp_out = 0; for (int l = 0; l < L; l++) limbs_out[l] = 0; return; }
    auto at = [&](int64_t l) -> uint64_t { return (l >= 0 && l < n) ? mag[l] : 0ull; };
    auto bits64 = [&](int64_t pos) -> uint64_t {
        if (pos <= -64) return 0;
        if (pos < 0) return at(0) << (-pos);
        const int64_t li = pos >> 6; const int bo = (int)(pos & 63);
        return bo ? ((at(li) >> bo) | (at(li + 1) << (64 - bo))) : at(li);
    };
    int64_t E = e_lsb + bl;
    const int64_t base = (int64_t)bl - 64 * L;
    const int drop = 64 * L - prec;
    const int64_t rpos = (int64_t)bl - prec - 1;
    int rbit = 0, sticky = 0;
    if (rpos >= 0) {
        rbit = (int)((at(rpos >> 6) >> (rpos & 63)) & 1);
        for (int64_t l = 0; l < (rpos >> 6) && !sticky; l++) if (at(l)) sticky = 1;
        if (!sticky && (rpos & 63) && (at(rpos >> 6) & ((1ull << (rpos & 63)) - 1))) sticky = 1;
    }
    const uint64_t w0 = bits64(base) & (drop ? ~((1ull << drop) - 1) : ~0ull);
    const bool up = rbit && (sticky || ((w0 >> drop) & 1));
    if (up) {
        bool allones = (w0 | ((1ull << drop) - 1)) == ~0ull;
        for (int l = 1; l < L && allones; l++) allones = bits64(base + 64 * l) == ~0ull;
        if (allones) {
            for (int l = 0; l < L - 1; l++) limbs_out[l] = 0;
            limbs_out[L - 1] = 1ull << 63;
            *sign_out = neg; *exp_out = E + 1;
            return;
        }
    }
    uint64_t c = up ? (1ull << drop) : 0ull;
    for (int l = 0; l < L; l++) {
        const uint64_t w = l == 0 ? w0 : bits64(base + 64 * l);
        const uint64_t x = w + c;
        c = x < w;
        limbs_out[l] = x;
    }
    *sign_out = neg; *exp_out = E;
}

constexpr int kF64Lmax = 80;      // fixed-point limbs: b (s + 1) + 64 <= 64 * 78 (prec <= 4096)

__global__ void __launch_bounds__(128)
fold_f64_kernel(const int64_t *__restrict__ partials, int64_t m, int64_t n, int s, int b, int method, int prec, int L,
                const int64_t *__restrict__ eA, const int64_t *__restrict__ eB, DMatOut Cre, DMatOut Cim)
{
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    for (int64_t i = blockIdx.y; i < m; i += gridDim.y) {
    const int64_t plane = m * n, off = i * n + j;
    uint64_t fix[2][kF64Lmax];
    const int Lc = (int)(((int64_t)b * (s + 1) + 64) / 64 + 1);
    for (int p = 0; p < 2; p++) for (int l = 0; l < Lc; l++) fix[p][l] = 0;
    int64_t carry[2] = {0, 0};
    const uint64_t mask = (1ull << b) - 1;
    int64_t bitpos = 0;                                   // of the next emitted digit
    for (int r = s + 1; r >= 2; r--) {
        int64_t t[3];
        for (int q = 0; q < 3; q++) t[q] = __ldg(partials + (int64_t)(q * (s + 2) + r) * plane + off);
        int64_t d[2];
        if (method == 3) { d[0] = t[0] - t[1]; d[1] = t[2] - t[0] - t[1]; }   // Eq. 6
        else             { d[0] = t[0] - t[1]; d[1] = t[2]; }                 // Eq. 5
        for (int p = 0; p < 2; p++) {
            carry[p] += d[p];
            const uint64_t dig = (uint64_t)carry[p] & mask;
            carry[p] >>= b;                                               // arithmetic
            const int li = (int)(bitpos >> 6), bo = (int)(bitpos & 63);
            fix[p][li] |= dig << bo;
            if (bo + b > 64) fix[p][li + 1] |= dig >> (64 - bo);
        }
        bitpos += b;
    }
    for (int p = 0; p < 2; p++) {                         // final carry at bit b s, sign-extended
        const int li = (int)(bitpos >> 6), bo = (int)(bitpos & 63);
        const uint64_t c = (uint64_t)carry[p], sx = carry[p] < 0 ? ~0ull : 0ull;
        fix[p][li] |= c << bo;
        if (li + 1 < Lc) fix[p][li + 1] = bo ? ((c >> (64 - bo)) | (sx << bo)) : sx;
        for (int l = li + 2; l < Lc; l++) fix[p][l] = sx;
    }
    const int64_t e0 = eA[i] + eB[j] + 6 - (int64_t)b * (s + 1);
    DMatOut *outs[2] = {&Cre, &Cim};
    for (int p = 0; p < 2; p++) {
        const bool neg = (int64_t)fix[p][Lc - 1] < 0;
        if (neg) { uint64_t c = 1; for (int l = 0; l < Lc; l++) { const uint64_t x = ~fix[p][l] + c; c = (c && x == 0); fix[p][l] = x; } }
        const int64_t o = i * outs[p]->ld + j;
        round_store_local(fix[p], Lc, e0, neg, prec, L, outs[p]->sign + o, outs[p]->exp + o, outs[p]->limbs + o * L);
    }
    }                                                     // rows i (grid-stride over gridDim.y)
}

cudaError_t fold_f64_launch(const int64_t *partials, int64_t m, int64_t n, int s, int b, int method, int prec, int L,
                            const int64_t *eA, const int64_t *eB, DMatOut Cre, DMatOut Cim, cudaStream_t st)
{
    if (m == 0 || n == 0) return cudaSuccess;
    if ((int64_t)b * (s + 1) + 64 > 64 * (kF64Lmax - 2)) return cudaErrorInvalidValue;
    dim3 grid((unsigned)((n + 127) / 128), (unsigned)(m < 65535 ? m : 65535));
    fold_f64_kernel<<<grid, 128, 0, st>>>(partials, m, n, s, b, method, prec, L, eA, eB, Cre, Cim);
    return cudaGetLastError();
}

}  // namespace mpc
