// stages.cu -- the HBM-bound steps of the hot path (sm_100a):
//   a-1 linemax          per-row / per-column max exponent (mu of Algorithm 2)
//   a-2 prepass_*        the rho-hat pre-pass planes and reductions
//   a-3 split            error-free split into balanced radix-256 digit planes
//   a-5/a-6 fold_normalize  exact fold of the slice products with the Eq. 5/6
//                        combination, carry propagation and one RNE rounding
#include <climits>
#include "common.cuh"
#include "kernels.h"

namespace mpc {

// limb idx of mantissa N (zero outside [0, L))
MPC_DEV uint64_t limb_at(const uint64_t *N, int L, int64_t idx) {
    return (idx >= 0 && idx < L) ? __ldg(N + idx) : 0ull;
}

// 64 bits of a little-endian limb array starting at bit pos (bits outside are zero)
MPC_DEV uint64_t bits64(const uint64_t *a, int n, int64_t pos) {
    if (pos <= -64) return 0;
    if (pos < 0) return (n > 0 ? a[0] : 0ull) << (-pos);
    int64_t li = pos >> 6;
    int bo = (int)(pos & 63);
    uint64_t lo = li < n ? a[li] : 0ull;
    if (!bo) return lo;
    uint64_t hi = li + 1 < n ? a[li + 1] : 0ull;
    return (lo >> bo) | (hi << (64 - bo));
}

// ================================================================== a-1: exponent scan
MPC_DEV uint64_t enc_exp(int64_t e) { return (uint64_t)e ^ 0x8000000000000000ull; }   // order-preserving

__global__ void linemax_kernel(DMat re, DMat im, int64_t rows, int64_t cols, int L, int prec, int side,
                               unsigned long long *emax, uint32_t *errflag, int validate)
{
    __shared__ unsigned long long red[8][33];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int64_t c = (int64_t)blockIdx.x * 32 + tx;
    unsigned long long colmax = 0;
    const uint64_t lowmask = (64 * L - prec) ? ((1ull << (64 * L - prec)) - 1) : 0ull;
    for (int64_t r = (int64_t)blockIdx.y * 8 + ty; r < rows; r += (int64_t)gridDim.y * 8) {
        unsigned long long v = 0;
        if (c < cols) {
#pragma unroll
            for (int p = 0; p < 2; p++) {
                const DMat &M = p ? im : re;
                const int64_t idx = r * M.ld + c;
                const uint64_t *N = M.limbs + idx * L;
                const uint64_t top = __ldg(N + L - 1);
                const int64_t e = __ldg(M.exp + idx);
                if (validate) {
                    uint32_t bad = 0;
                    if (top) {
                        if (!(top >> 63)) bad |= 1u;
                        if (__ldg(N) & lowmask) bad |= 1u;
                        if (e > (1ll << 61) || e < -(1ll << 61)) bad |= 2u;
                    } else {
                        for (int l = 0; l < L - 1; l++) if (__ldg(N + l)) bad |= 1u;
                    }
                    if (bad) atomicOr(errflag, bad);
                }
                if (top) { unsigned long long x = enc_exp(e); v = x > v ? x : v; }
            }
        }
        if (side == 0) {
            // reduce over the 32 columns of this warp (one row)
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                unsigned long long y = __shfl_xor_sync(0xffffffffu, v, o);
                v = y > v ? y : v;
            }
            if (tx == 0 && v) atomicMax(&emax[r], v);
        } else {
            colmax = v > colmax ? v : colmax;
        }
    }
    if (side == 1) {
        red[ty][tx] = colmax;
        __syncthreads();
        if (ty == 0 && c < cols) {
            unsigned long long v = red[0][tx];
            for (int y = 1; y < 8; y++) v = red[y][tx] > v ? red[y][tx] : v;
            if (v) atomicMax(&emax[c], v);
        }
    }
}

__global__ void linemax_finalize_kernel(unsigned long long *emax, int64_t n, int64_t *eline, uint8_t *nz) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    unsigned long long v = emax[i];
    nz[i] = v ? 1 : 0;
    eline[i] = v ? (int64_t)(v ^ 0x8000000000000000ull) : 0;
}

cudaError_t linemax_launch(DMat re, DMat im, int64_t rows, int64_t cols, int L, int prec, int side,
                           int64_t *eline, uint8_t *nz, uint32_t *errflag, int validate, cudaStream_t st)
{
    const int64_t lines = side == 0 ? rows : cols;
    if (lines == 0) return cudaSuccess;
    // eline doubles as the encoded accumulator (same 8-byte slots)
    unsigned long long *acc = reinterpret_cast<unsigned long long *>(eline);
    cudaError_t e = cudaMemsetAsync(acc, 0, sizeof(unsigned long long) * lines, st);
    if (e != cudaSuccess) return e;
    if (rows > 0 && cols > 0) {
        dim3 block(32, 8);
        int64_t gy = (rows + 7) / 8;
        if (side == 1) gy = gy < 64 ? gy : 64;
        else gy = gy < 65535 ? gy : 65535;
        dim3 grid((unsigned)((cols + 31) / 32), (unsigned)gy);
        linemax_kernel<<<grid, block, 0, st>>>(re, im, rows, cols, L, prec, side, acc, errflag, validate);
    }
    linemax_finalize_kernel<<<(unsigned)((lines + 255) / 256), 256, 0, st>>>(acc, lines, eline, nz);
    return cudaGetLastError();
}

// ================================================================== a-3: split into digit planes
// Streams the bytes of X = floor(N 2^(W - e + exp - 64L)) from the least significant one:
// byte t of X = bits [pos0 + 8t, pos0 + 8t + 8) of N, pos0 = 64L - W + e - exp.
struct ByteStream {
    const uint64_t *N;
    int L;
    int64_t pos;     // bit position of the next byte
    int64_t li;      // cached limb index
    uint64_t lo, hi;
    MPC_DEV void init(const uint64_t *N_, int L_, int64_t pos0, bool zero) {
        N = N_; L = zero ? 0 : L_; pos = pos0;
        li = pos >= 0 ? (pos >> 6) : -((-pos + 63) >> 6);
        lo = limb_at(N, L, li); hi = limb_at(N, L, li + 1);
    }
    MPC_DEV uint32_t next() {
        const int64_t l = pos >= 0 ? (pos >> 6) : -((-pos + 63) >> 6);   // floor(pos / 64)
        if (l != li) {
            if (l == li + 1) { lo = hi; hi = limb_at(N, L, l + 1); }
            else { lo = limb_at(N, L, l); hi = limb_at(N, L, l + 1); }
            li = l;
        }
        const int bo = (int)(pos - (l << 6));
        uint64_t v = bo ? ((lo >> bo) | (hi << (64 - bo))) : lo;
        pos += 8;
        return (uint32_t)(v & 0xFF);
    }
};

__global__ void split_kernel(DMat re, DMat im, int side, int64_t lines, int64_t k, int64_t kp, int L,
                             const int64_t *__restrict__ eline, int s, int nparts, int8_t *__restrict__ dig)
{
    const int64_t kk = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (kk >= kp) return;
    const int64_t plane = lines * kp;
    for (int64_t line = blockIdx.y; line < lines; line += gridDim.y) {
        int8_t *out = dig + line * kp + kk;
        if (kk >= k) {
            for (int a = 0; a < nparts * s; a++) out[(int64_t)a * plane] = 0;
            continue;
        }
        const int64_t e = eline[line];
        const int64_t W = 8 * (int64_t)s - 3;
        ByteStream bs[2];
        uint32_t neg[2], nc[2];
#pragma unroll
        for (int p = 0; p < 2; p++) {
            const DMat &M = p ? im : re;
            const int64_t idx = side == 0 ? line * M.ld + kk : kk * M.ld + line;
            const uint64_t *N = M.limbs + idx * L;
            const bool zero = __ldg(N + L - 1) == 0;
            const int64_t ex = __ldg(M.exp + idx);
            bs[p].init(N, L, 64 * (int64_t)L - W + e - ex, zero);
            neg[p] = zero ? 0u : (uint32_t)__ldg(M.sign + idx);
            nc[p] = 1;                              // +1 of the two's complement negation
        }
        uint32_t csum = 0;                          // carry of the 3M byte-stream addition
        uint32_t rc[3] = {0, 0, 0};                 // balanced-recoding carries
        for (int t = 0; t < s; t++) {
            uint32_t y[3];
#pragma unroll
            for (int p = 0; p < 2; p++) {
                uint32_t b = bs[p].next();
                if (neg[p]) { uint32_t v = (~b & 0xFFu) + nc[p]; nc[p] = v >> 8; b = v & 0xFFu; }
                y[p] = b;
            }
            {
                uint32_t v = y[0] + y[1] + csum;
                csum = v >> 8; y[2] = v & 0xFFu;
            }
            const int64_t a = s - 1 - t;            // plane of digit alpha = s - t
#pragma unroll
            for (int p = 0; p < 3; p++) {
                if (p < nparts) {
                    uint32_t v = y[p] + rc[p];
                    int d = v >= 128u ? (int)v - 256 : (int)v;
                    rc[p] = v >= 128u;
                    out[((int64_t)p * s + a) * plane] = (int8_t)d;
                }
            }
        }
    }
}

cudaError_t split_launch(DMat re, DMat im, int side, int64_t lines, int64_t k, int64_t kp, int L,
                         const int64_t *eline, int s, int nparts, int8_t *dig, cudaStream_t st)
{
    if (lines == 0 || kp == 0) return cudaSuccess;
    dim3 grid((unsigned)((kp + 127) / 128), (unsigned)(lines < 65535 ? lines : 65535));
    split_kernel<<<grid, 128, 0, st>>>(re, im, side, lines, k, kp, L, eline, s, nparts, dig);
    return cudaGetLastError();
}

// ================================================================== a-2: pre-pass
// relative entry exponents for the max-plus stage: real entries clamped to [-2^28, 0], zero
// entries -2^30, so a sum is > -2^30 iff both entries are nonzero (no int32 overflow:
// sentinel + sentinel = -2^31)
constexpr int32_t kRelSentinel = -(1 << 30);
constexpr int32_t kRelClamp = -(1 << 28);

__global__ void prepass_planes_kernel(DMat re, DMat im, int side, int64_t lines, int64_t k, int64_t kp, int L,
                                      const int64_t *__restrict__ eline, int8_t *t, int32_t *rel)
{
    const int64_t kk = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (kk >= kp) return;
    for (int64_t line = blockIdx.y; line < lines; line += gridDim.y) {
        int best = 0;
        int64_t emax = 0; bool any = false;
        if (kk < k) {
            const int64_t e = eline[line];
#pragma unroll
            for (int p = 0; p < 2; p++) {
                const DMat &M = p ? im : re;
                const int64_t idx = side == 0 ? line * M.ld + kk : kk * M.ld + line;
                const uint64_t *N = M.limbs + idx * L;
                const uint64_t top = __ldg(N + L - 1);
                if (!top) continue;
                const int64_t ex = __ldg(M.exp + idx);
                // t = floor(|x| 2^(7-e)) = bits [64L - 7 + e - ex, 64L) of N
                const int64_t pos = 64 * (int64_t)L - 7 + e - ex;
                uint64_t v = 0;
                if (pos < 64 * (int64_t)L) {
                    const int64_t li = pos >> 6;
                    const int bo = (int)(pos & 63);
                    const uint64_t lo = __ldg(N + li);
                    const uint64_t hi = li + 1 < L ? __ldg(N + li + 1) : 0ull;
                    v = bo ? ((lo >> bo) | (hi << (64 - bo))) : lo;
                }
                int tv = (int)(v & 0x7F);
                best = tv > best ? tv : best;
                if (!any || ex > emax) emax = ex;
                any = true;
            }
        }
        t[line * kp + kk] = (int8_t)best;
        int32_t r = kRelSentinel;
        if (any) {
            int64_t d = emax - eline[line];         // <= 0
            r = d < kRelClamp ? kRelClamp : (int32_t)d;
        }
        rel[line * kp + kk] = r;
    }
}

cudaError_t prepass_planes_launch(DMat re, DMat im, int side, int64_t lines, int64_t k, int64_t kp, int L,
                                  const int64_t *eline, int8_t *t, int32_t *rel, cudaStream_t st)
{
    if (lines == 0 || kp == 0) return cudaSuccess;
    dim3 grid((unsigned)((kp + 127) / 128), (unsigned)(lines < 65535 ? lines : 65535));
    prepass_planes_kernel<<<grid, 128, 0, st>>>(re, im, side, lines, k, kp, L, eline, t, rel);
    return cudaGetLastError();
}

MPC_DEV int64_t sum_T(const int32_t *T, int nslots, int64_t plane, int64_t off) {
    int64_t v = 0;
    for (int q = 0; q < nslots; q++) v += T[(int64_t)q * plane + off];
    return v;
}

// stage 1: min over nonzero line pairs of T_ij
__global__ void prepass_min_kernel(const int32_t *T, int nslots, int64_t plane, int64_t ldD, int64_t m, int64_t n,
                                   const uint8_t *nzA, const uint8_t *nzB, unsigned long long *out_min)
{
    unsigned long long best = ULLONG_MAX;
    const int64_t total = m * n;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / n, j = t - i * n;
        if (!nzA[i] || !nzB[j]) continue;
        const unsigned long long v = (unsigned long long)sum_T(T, nslots, plane, i * ldD + j);
        best = v < best ? v : best;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        unsigned long long y = __shfl_xor_sync(0xffffffffu, best, o);
        best = y < best ? y : best;
    }
    if ((threadIdx.x & 31) == 0 && best != ULLONG_MAX) atomicMin(out_min, best);
}

// stage 2: exact max-plus exponent bound and the per-pair bound choice
__global__ void __launch_bounds__(256)
prepass_maxplus_kernel(const int32_t *T, int nslots, int64_t plane, int64_t ldD, int64_t m, int64_t n,
                       int64_t k, int64_t kp, const uint8_t *nzA, const uint8_t *nzB,
                       const int32_t *relA, const int32_t *relB,
                       unsigned long long *out_min, unsigned long long *out_min1, long long *out_max2)
{
    __shared__ int32_t sa[32][33], sb[32][33];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;    // 32 x 8
    const int64_t i0 = (int64_t)blockIdx.y * 32, j0 = (int64_t)blockIdx.x * 32;
    int32_t mp[4] = {kRelSentinel, kRelSentinel, kRelSentinel, kRelSentinel};
    for (int64_t k0 = 0; k0 < k; k0 += 32) {
        __syncthreads();
        for (int q = threadIdx.x; q < 32 * 32; q += 256) {
            const int rr = q >> 5, cc = q & 31;
            const int64_t kk = k0 + cc;
            sa[rr][cc] = (i0 + rr < m && kk < k) ? relA[(i0 + rr) * kp + kk] : kRelSentinel;
            sb[rr][cc] = (j0 + rr < n && kk < k) ? relB[(j0 + rr) * kp + kk] : kRelSentinel;
        }
        __syncthreads();
#pragma unroll
        for (int e = 0; e < 4; e++) {
            int32_t best = mp[e];
            const int r_ = ty * 4 + e;
#pragma unroll 8
            for (int cc = 0; cc < 32; cc++) { int32_t x = sa[r_][cc] + sb[tx][cc]; best = x > best ? x : best; }
            mp[e] = best;
        }
    }
    unsigned long long lmin = ULLONG_MAX, lmin1 = ULLONG_MAX;
    long long lmax2 = -1;
    for (int e = 0; e < 4; e++) {
        const int64_t i = i0 + ty * 4 + e, j = j0 + tx;
        if (i >= m || j >= n || !nzA[i] || !nzB[j]) continue;
        if (mp[e] <= kRelSentinel) continue;                // no common support: (|A||B|)_ij = 0
        const int64_t Tv = sum_T(T, nslots, plane, i * ldD + j);
        const int64_t D = -(int64_t)mp[e];
        lmin = (unsigned long long)Tv < lmin ? (unsigned long long)Tv : lmin;
        const bool use2 = (Tv == 0) || (D < 12 && (Tv << D) < 4096);
        if (use2) lmax2 = D > lmax2 ? D : lmax2;
        else lmin1 = (unsigned long long)Tv < lmin1 ? (unsigned long long)Tv : lmin1;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        unsigned long long y = __shfl_xor_sync(0xffffffffu, lmin, o); lmin = y < lmin ? y : lmin;
        y = __shfl_xor_sync(0xffffffffu, lmin1, o); lmin1 = y < lmin1 ? y : lmin1;
        long long z = __shfl_xor_sync(0xffffffffu, lmax2, o); lmax2 = z > lmax2 ? z : lmax2;
    }
    if (tx == 0) {
        if (lmin != ULLONG_MAX) atomicMin(out_min, lmin);
        if (lmin1 != ULLONG_MAX) atomicMin(out_min1, lmin1);
        if (lmax2 >= 0) atomicMax(out_max2, lmax2);
    }
}

cudaError_t prepass_reduce_launch(const int32_t *T, int nslots, int64_t plane, int64_t ldD,
                                  int64_t m, int64_t n, int64_t k, int64_t kp,
                                  const uint8_t *nzA, const uint8_t *nzB, const int32_t *relA, const int32_t *relB,
                                  int stage, unsigned long long *out_min, unsigned long long *out_min1,
                                  long long *out_max2, cudaStream_t st)
{
    if (m == 0 || n == 0) return cudaSuccess;
    if (stage == 1) {
        int64_t blocks = (m * n + 255) / 256;
        if (blocks > 148 * 16) blocks = 148 * 16;
        prepass_min_kernel<<<(unsigned)blocks, 256, 0, st>>>(T, nslots, plane, ldD, m, n, nzA, nzB, out_min);
    } else {
        dim3 grid((unsigned)((n + 31) / 32), (unsigned)((m + 31) / 32));
        prepass_maxplus_kernel<<<grid, 256, 0, st>>>(T, nslots, plane, ldD, m, n, k, kp, nzA, nzB, relA, relB,
                                                     out_min, out_min1, out_max2);
    }
    return cudaGetLastError();
}

// ================================================================== a-5 + a-6: fold and normalize
constexpr int kLcMax = kMaxSlices / 8 + 4;

// two's complement fix[0..Lc) -> RNE to prec bits in the ABI format
MPC_DEV void normalize_store(uint64_t *fix, int Lc, int64_t e0, int prec, int L,
                             uint8_t *sign_out, int64_t *exp_out, uint64_t *limbs_out)
{
    const bool neg = (int64_t)fix[Lc - 1] < 0;
    if (neg) {                                        // magnitude
        uint64_t c = 1;
        for (int l = 0; l < Lc; l++) { uint64_t x = ~fix[l] + c; c = (c && x == 0); fix[l] = x; }
    }
    int b = 0;
    for (int l = Lc - 1; l >= 0; l--)
        if (fix[l]) { b = 64 * l + 64 - __clzll((long long)fix[l]); break; }
    if (b == 0) {
        *sign_out = 0; *exp_out = 0;
        for (int l = 0; l < L; l++) limbs_out[l] = 0;
        return;
    }
    int64_t E = e0 + b;
    // top-aligned window of 64L bits ending at bit b
    uint64_t out[64];
    const int64_t base = (int64_t)b - 64 * L;
    for (int l = 0; l < L; l++) out[l] = bits64(fix, Lc, base + 64 * l);
    const int drop = 64 * L - prec;                   // low bits of the window below prec
    // round bit = bit (b - prec - 1) of the magnitude; sticky = any lower bit
    const int64_t rpos = (int64_t)b - prec - 1;
    int rbit = 0, sticky = 0;
    if (rpos >= 0) {
        rbit = (int)((fix[rpos >> 6] >> (rpos & 63)) & 1);
        const int64_t full = rpos >> 6;
        for (int64_t l = 0; l < full && !sticky; l++) if (fix[l]) sticky = 1;
        if (!sticky && (rpos & 63)) if (fix[full] & ((1ull << (rpos & 63)) - 1)) sticky = 1;
    }
    if (drop) out[0] &= ~((1ull << drop) - 1);
    const int lsb = (int)((out[0] >> drop) & 1);
    if (rbit && (sticky || lsb)) {
        uint64_t c = 1ull << drop;
        for (int l = 0; l < L && c; l++) { uint64_t x = out[l] + c; c = x < out[l] ? 1 : 0; out[l] = x; }
        if (c) {                                      // carry-out: 2^prec -> 2^(prec-1)
            for (int l = 0; l < L; l++) out[l] = 0;
            out[L - 1] = 1ull << 63;
            E += 1;
        }
    }
    *sign_out = neg ? 1 : 0;
    *exp_out = E;
    for (int l = 0; l < L; l++) limbs_out[l] = out[l];
}

__global__ void __launch_bounds__(128)
fold_normalize_kernel(const FoldParams F)
{
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t i = blockIdx.y;
    if (j >= F.n || i >= F.m) return;
    const int s = F.s;
    const int Lc = s / 8 + 3;
    uint64_t fix[2][kLcMax];
    uint64_t cur[2] = {0, 0};
    int64_t carry[2] = {0, 0};
    const int64_t off = i * F.ldD + j;
    for (int r = s + 1; r >= 2; r--) {
        int64_t t[kMaxJobs];
#pragma unroll
        for (int q = 0; q < kMaxJobs; q++) {
            const int base = F.slotinfo[(q * (s + 2) + r) * 2], cnt = F.slotinfo[(q * (s + 2) + r) * 2 + 1];
            int64_t v = 0;
            for (int c = 0; c < cnt; c++) v += __ldg(F.partials + (int64_t)(base + c) * F.plane + off);
            t[q] = v;
        }
        int64_t d[2];
        if (F.method == 3) { d[0] = t[0] - t[1]; d[1] = t[2] - t[0] - t[1]; }   // Eq. 6
        else               { d[0] = t[0] - t[1]; d[1] = t[2]; }                 // Eq. 5
        const int b = s + 1 - r;                                                // byte index
#pragma unroll
        for (int p = 0; p < 2; p++) {
            carry[p] += d[p];
            cur[p] |= (uint64_t)(carry[p] & 0xFF) << (8 * (b & 7));
            carry[p] >>= 8;                                                     // arithmetic
            if ((b & 7) == 7) { fix[p][b >> 3] = cur[p]; cur[p] = 0; }
        }
    }
    // append the final carry at bit 8s, sign-extended
    const int l0 = s >> 3, o = 8 * (s & 7);
#pragma unroll
    for (int p = 0; p < 2; p++) {
        const uint64_t c = (uint64_t)carry[p];
        const uint64_t sext = carry[p] < 0 ? ~0ull : 0ull;
        fix[p][l0] = cur[p] | (c << o);
        fix[p][l0 + 1] = o ? ((c >> (64 - o)) | (sext << o)) : sext;
        for (int l = l0 + 2; l < Lc; l++) fix[p][l] = sext;
    }
    const int64_t e0 = F.eA[i] + F.eB[j] + 6 - 8 * (int64_t)(s + 1);
    const int64_t oi = i * F.Cre.ld + j;
    normalize_store(fix[0], Lc, e0, F.prec, F.L, F.Cre.sign + oi, F.Cre.exp + oi, F.Cre.limbs + oi * F.L);
    const int64_t oj = i * F.Cim.ld + j;
    normalize_store(fix[1], Lc, e0, F.prec, F.L, F.Cim.sign + oj, F.Cim.exp + oj, F.Cim.limbs + oj * F.L);
}

cudaError_t fold_normalize_launch(const FoldParams &F, cudaStream_t st)
{
    if (F.m == 0 || F.n == 0) return cudaSuccess;
    if (F.s > kMaxSlices) return cudaErrorInvalidValue;
    dim3 grid((unsigned)((F.n + 127) / 128), (unsigned)F.m);
    fold_normalize_kernel<<<grid, 128, 0, st>>>(F);
    return cudaGetLastError();
}

__global__ void zero_output_kernel(DMatOut C, int64_t m, int64_t n, int L) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t i = blockIdx.y;
    if (j >= n) return;
    const int64_t o = i * C.ld + j;
    C.sign[o] = 0; C.exp[o] = 0;
    for (int l = 0; l < L; l++) C.limbs[o * L + l] = 0;
}

cudaError_t zero_output_launch(DMatOut C, int64_t m, int64_t n, int L, cudaStream_t st) {
    if (m == 0 || n == 0) return cudaSuccess;
    dim3 grid((unsigned)((n + 127) / 128), (unsigned)m);
    zero_output_kernel<<<grid, 128, 0, st>>>(C, m, n, L);
    return cudaGetLastError();
}

}  // namespace mpc
