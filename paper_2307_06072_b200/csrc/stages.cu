// stages.cu -- the HBM-bound steps of the hot path (sm_100a):
//   a-1 linemax          per-row / per-column max exponent (mu of Algorithm 2)
//   a-2 prepass_*        the rho-hat pre-pass planes and reductions
//   a-3 split            error-free split into balanced radix-256 digit planes
//   a-5/a-6 fold_normalize  exact fold of the slice products with the Eq. 5/6
//                        combination, carry propagation and one RNE rounding
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cuda.h>
#include "common.cuh"
#include "kernels.h"
#include "rule.cuh"

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

// block (bx, by) of a (., gy) grid over one side
// tb (or null): the entries' top bytes for the pre-pass planes, tb[part * tbpart + (tbline0 + line) * tbkp + kk]
// = max(1, top limb >> 56) for a nonzero entry, 0 for zero -- the planes then read these bytes and the
// contiguous exponents instead of one 32-byte sector of every 8L-byte entry (t depends only on the top
// byte: t = top >> (57 + e - ex) and e - ex <= 6 where it is nonzero)
MPC_DEV void linemax_body(const DMat &re, const DMat &im, int64_t rows, int64_t cols, int L, int prec, int side,
                          unsigned long long *emax, uint32_t *errflag, int validate, int64_t bx, int64_t by, int64_t gy,
                          uint8_t *tb = nullptr, int64_t tbkp = 0, int64_t tbline0 = 0, int64_t tbpart = 0)
{
    __shared__ unsigned long long red[8][33];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int64_t c = bx * 32 + tx;
    unsigned long long colmax = 0;
    const uint64_t lowmask = (64 * L - prec) ? ((1ull << (64 * L - prec)) - 1) : 0ull;
    for (int64_t r = by * 8 + ty; r < rows; r += gy * 8) {
        unsigned long long v = 0;
        if (c < cols) {
#pragma unroll
            for (int p = 0; p < 2; p++) {
                const DMat &M = p ? im : re;
                const int64_t idx = r * M.ld + c;
                const uint64_t *N = M.limbs + idx * L;
                const uint64_t top = __ldg(N + L - 1);
                const int64_t e = __ldg(M.exp + idx);
                if (tb) {
                    const uint64_t hb = top >> 56;
                    const uint8_t b = top ? (uint8_t)(hb ? hb : 1ull) : (uint8_t)0;
                    tb[p * tbpart + (tbline0 + (side ? c : r)) * tbkp + (side ? r : c)] = b;
                }
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

__global__ void linemax_kernel(DMat re, DMat im, int64_t rows, int64_t cols, int L, int prec, int side,
                               unsigned long long *emax, uint32_t *errflag, int validate)
{
    linemax_body(re, im, rows, cols, L, prec, side, emax, errflag, validate, blockIdx.x, blockIdx.y, gridDim.y);
}

// both sides in one launch: blocks [0, gx0*gy0) scan the rows of A, the rest the columns of B.
// The last block to finish (a done counter zeroed with the accumulators) decodes the maxima
// in place into eline / nz (the finalize step, without a launch of its own)
__global__ void linemax2_kernel(DMat re0, DMat im0, int64_t rows0, int64_t cols0, DMat re1, DMat im1, int64_t rows1,
                                int64_t cols1, int L, int prec, unsigned long long *emax0, unsigned long long *emax1,
                                uint32_t *errflag, int validate, int64_t gx0, int64_t gy0, int64_t gx1, int64_t gy1,
                                unsigned int *done, int64_t *eline, uint8_t *nz, int64_t lines, int clean, uint8_t *tb,
                                int64_t tbkp)
{
    pdl_wait();
    const int64_t b = blockIdx.x;
    if (b < gx0 * gy0)
        linemax_body(re0, im0, rows0, cols0, L, prec, 0, emax0, errflag, validate, b % gx0, b / gx0, gy0, tb, tbkp, 0,
                     lines * tbkp);
    else {
        const int64_t c = b - gx0 * gy0;
        linemax_body(re1, im1, rows1, cols1, L, prec, 1, emax1, errflag, validate, c % gx1, c / gx1, gy1, tb, tbkp, rows0,
                     lines * tbkp);
    }
    __shared__ int last;
    const int tid = threadIdx.y * blockDim.x + threadIdx.x;
    __syncthreads();                                  // this block's atomics issued
    if (tid == 0) { __threadfence(); last = atomicAdd(done, 1u) == gridDim.x - 1; }
    __syncthreads();
    if (!last) return;
    __threadfence();
    unsigned long long *acc = emax0;                  // emax0 .. emax0 + lines (eA then eB)
    for (int64_t i = tid; i < lines; i += (int64_t)blockDim.x * blockDim.y) {
        const unsigned long long v = __ldcg(acc + i);
        nz[i] = v ? 1 : 0;
        eline[i] = v ? (int64_t)(v ^ 0x8000000000000000ull) : 0;
        if (clean) acc[i] = 0;                        // separate accumulators: zero them (and the done
    }                                                 // counter) for the next call -- no memset node
    if (clean && tid == 0) *done = 0;
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

// a-1 for A (rows) and B (columns) together: one accumulator memset (eA, eB contiguous), one scan
// launch, one finalize launch (nz and eline of both sides contiguous too)
cudaError_t linemax2_launch(DMat Are, DMat Aim, DMat Bre, DMat Bim, int64_t m, int64_t n, int64_t k, int L, int prec,
                            int64_t *eAB, uint8_t *nzAB, uint32_t *errflag, int validate, cudaStream_t st, int *nlaunch,
                            unsigned long long *acc_clean, uint8_t *tb, int64_t tbkp)
{
    if (nlaunch) *nlaunch = 0;
    if (m + n == 0) return cudaSuccess;
    const int64_t gx0 = m > 0 ? (k + 31) / 32 : 0, gy0 = std::min<int64_t>((m + 7) / 8, 65535);
    const int64_t gx1 = n > 0 ? (n + 31) / 32 : 0, gy1 = std::min<int64_t>((k + 7) / 8, 64);
    const int64_t blocks = k > 0 ? gx0 * gy0 + gx1 * gy1 : 0;
    unsigned long long *acc = reinterpret_cast<unsigned long long *>(eAB);
    unsigned int *done;
    const int clean = acc_clean && blocks > 0;
    if (clean) {
        // caller-kept accumulators (m + n words, then the done counter), all zero on entry; the
        // last block zeroes them again after the decode
        acc = acc_clean;
        done = reinterpret_cast<unsigned int *>(acc_clean + m + n);
    } else {
        // the accumulators, nz (overwritten by the decode) and the done counter after nz (8-aligned;
        // the metadata layout leaves >= 64 bytes there) in one memset
        done = reinterpret_cast<unsigned int *>((reinterpret_cast<uintptr_t>(nzAB + m + n) + 7) & ~uintptr_t(7));
        cudaError_t e = cudaMemsetAsync(acc, 0, reinterpret_cast<uint8_t *>(done + 2) - reinterpret_cast<uint8_t *>(acc), st);
        if (e != cudaSuccess) return e;
    }
    if (blocks > 0) {
        const cudaError_t le = launch_pdl(linemax2_kernel, dim3((unsigned)blocks), dim3(32, 8), 0, st, Are, Aim, m, k, Bre,
                                          Bim, k, n, L, prec, acc, acc + m, errflag, validate, gx0, gy0, gx1, gy1, done,
                                          eAB, nzAB, m + n, clean, tb, tbkp);
        if (le != cudaSuccess) return le;
    } else {
        linemax_finalize_kernel<<<(unsigned)((m + n + 255) / 256), 256, 0, st>>>(acc, m + n, eAB, nzAB);
    }
    if (nlaunch) *nlaunch = 1;
    return cudaGetLastError();
}

// ================================================================== a-3: split into digit planes
// X = sign * floor(|x| 2^(W - e)), W = 8s - 3 (reading Z5), as a two's complement integer;
// its s balanced radix-256 digits (digit set [-128,127]) are the bytes of Z = X + H,
// H = sum_t 128 * 256^t, minus 128 (Z's bytes are the unique base-256 digits of X + H, and
// X + H = sum (d_t + 128) 256^t with d_t + 128 in [0,255]).  So the split is word arithmetic:
// funnel-shift the mantissa into 64-bit words of X, negate (two's complement) for x < 0, add
// Re + Im for the 3M sum part, add H with carry, and XOR 0x80 into every byte.
// Each thread handles VEC = 4 consecutive k of one line, so each digit-plane store is one
// coalesced 32-bit write.
struct WordStream {
    const uint64_t *N;
    int L;
    int64_t li;          // limb index of the low part of the next word
    int bo;              // bit offset inside it
    uint64_t lo;
    MPC_DEV void init(const uint64_t *N_, int L_, int64_t pos0, bool zero) {
        N = N_; L = zero ? 0 : L_;
        li = pos0 >= 0 ? (pos0 >> 6) : -((-pos0 + 63) >> 6);     // floor(pos0 / 64)
        bo = (int)(pos0 - (li << 6));
        lo = limb_at(N, L, li);
    }
    MPC_DEV uint64_t next() {
        const uint64_t hi = limb_at(N, L, li + 1);
        const uint64_t v = bo ? ((lo >> bo) | (hi << (64 - bo))) : lo;
        lo = hi; li++;
        return v;
    }
};

constexpr int kSplitVec = 4;
constexpr uint64_t kH = 0x8080808080808080ull;

__global__ void __launch_bounds__(128, 4)
split_kernel(DMat re, DMat im, int side, int64_t lines, int64_t k, int64_t kp, int L,
             const int64_t *__restrict__ eline, int s, int nparts, int8_t *__restrict__ dig, const DevRuleState *drs)
{
    if (drs) { if (drs->status) return; s = drs->cur.s; }    // device rule: the chosen s
    const int64_t kk0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * kSplitVec;
    if (kk0 >= kp) return;
    const int64_t plane = lines * kp;
    const int64_t W = 8 * (int64_t)s - 3;
    for (int64_t line = blockIdx.y; line < lines; line += gridDim.y) {
        const int64_t e = eline[line];
        WordStream ws[kSplitVec][2];
        uint64_t nc[kSplitVec][2];
        uint32_t neg[kSplitVec][2];
        uint64_t csum[kSplitVec];
        uint64_t ch[kSplitVec][3];
#pragma unroll
        for (int v = 0; v < kSplitVec; v++) {
            const int64_t kk = kk0 + v;
#pragma unroll
            for (int p = 0; p < 2; p++) {
                const DMat &M = p ? im : re;
                if (kk < k) {
                    const int64_t idx = side == 0 ? line * M.ld + kk : kk * M.ld + line;
                    const uint64_t *N = M.limbs + idx * L;
                    const bool zero = __ldg(N + L - 1) == 0;
                    const int64_t ex = __ldg(M.exp + idx);
                    ws[v][p].init(N, L, 64 * (int64_t)L - W + e - ex, zero);
                    neg[v][p] = zero ? 0u : (uint32_t)__ldg(M.sign + idx);
                } else {
                    ws[v][p].init(nullptr, 0, 0, true);
                    neg[v][p] = 0u;
                }
                nc[v][p] = 1;
            }
            csum[v] = 0;
            ch[v][0] = ch[v][1] = ch[v][2] = 0;
        }
        int8_t *out = dig + line * kp + kk0;
        const int nwords = (s + 7) / 8;
        for (int w = 0; w < nwords; w++) {
            uint64_t dw[3][kSplitVec];
#pragma unroll
            for (int v = 0; v < kSplitVec; v++) {
                uint64_t y[3];
#pragma unroll
                for (int p = 0; p < 2; p++) {
                    uint64_t x = ws[v][p].next();
                    if (neg[v][p]) { const uint64_t t = ~x + nc[v][p]; nc[v][p] = (nc[v][p] && t == 0) ? 1ull : 0ull; x = t; }
                    y[p] = x;
                }
                {   // 3M: Re + Im (two's complement, with carry)
                    const uint64_t t = y[0] + y[1];
                    const uint64_t c1 = t < y[0];
                    y[2] = t + csum[v];
                    csum[v] = c1 | (y[2] < t);
                }
#pragma unroll
                for (int p = 0; p < 3; p++) {            // + H with carry, XOR 0x80 per byte
                    const uint64_t t = y[p] + kH;
                    const uint64_t c1 = t < y[p];
                    const uint64_t z = t + ch[v][p];
                    ch[v][p] = c1 | (z < t);
                    dw[p][v] = z ^ kH;
                }
            }
            const int nb = min(8, s - 8 * w);
#pragma unroll
            for (int p = 0; p < 3; p++) {
                if (p >= nparts) break;
                for (int bt = 0; bt < nb; bt++) {
                    const int t = 8 * w + bt;            // digit t from the bottom -> plane s-1-t
                    uint32_t packed = 0;
#pragma unroll
                    for (int v = 0; v < kSplitVec; v++) packed |= (uint32_t)((dw[p][v] >> (8 * bt)) & 0xFF) << (8 * v);
                    *reinterpret_cast<uint32_t *>(out + ((int64_t)p * s + (s - 1 - t)) * plane) = packed;
                }
            }
        }
    }
}

// 64-bit add with carry-in c (0/1) and carry-out into c, as one PTX carry chain (the compiler's
// compare-based carries cost about twice the instructions; the split is issue-bound)
MPC_DEV uint64_t add64_carry(uint64_t a, uint64_t b, uint32_t &c) {
    uint32_t lo, hi, co;
    asm("{\n\t.reg .u32 t;\n\t"
        "add.cc.u32 t, %3, 0xFFFFFFFF;\n\t"      // CF = c
        "addc.cc.u32 %0, %4, %5;\n\t"
        "addc.cc.u32 %1, %6, %7;\n\t"
        "addc.u32 %2, 0, 0;\n\t}"
        : "=r"(lo), "=r"(hi), "=r"(co)
        : "r"(c), "r"((uint32_t)a), "r"((uint32_t)b), "r"((uint32_t)(a >> 32)), "r"((uint32_t)(b >> 32)));
    c = co;
    return ((uint64_t)hi << 32) | lo;
}

// bits [bo, bo + 64) of hi:lo (0 <= bo < 64) as two 32-bit funnel shifts of word pairs chosen by
// bo >= 32 (no 64-bit shift pair and no bo == 0 branch)
MPC_DEV uint64_t funnel64(uint64_t lo, uint64_t hi, uint32_t bo) {
    const uint32_t l0 = (uint32_t)lo, l1 = (uint32_t)(lo >> 32), h0 = (uint32_t)hi, h1 = (uint32_t)(hi >> 32);
    const bool up = bo >= 32;
    const uint32_t w0 = up ? l1 : l0, w1 = up ? h0 : l1, w2 = up ? h1 : h0;
    return ((uint64_t)__funnelshift_r(w1, w2, bo) << 32) | __funnelshift_r(w0, w1, bo);   // (shift mod 32)
}

// TMA-staged split (L in {2, 4, 8, 16}): a CTA takes kSplitT consecutive k of one line; one thread
// issues two 3-D TMA loads (Re, Im) of the 256 entries' limbs into shared memory -- coalesced,
// vectorised, every DRAM sector read once; the rows land swizzled (the swizzle span = one 8L-byte
// entry row) so that the per-word reads of consecutive entries by consecutive lanes spread over
// the banks -- while each thread loads its entry's exponent and sign.  Thread t then streams the
// words of entry k0 + t (same word arithmetic as split_kernel) and writes one byte per digit
// plane: a warp writes 32 consecutive bytes (one sector) of a plane row per store.
constexpr int kSplitT = 128;           // k per CTA = threads per CTA

// one CTA: kSplitT consecutive k of line `line` (k0 = first k); mre / mim: the tensor maps of the
// side's Re / Im limbs (kernel parameters)
template <int L, bool WS>
MPC_DEV void split_tma_body(const CUtensorMap *mre_p, const CUtensorMap *mim_p, const DMat &re, const DMat &im,
                            int side, int64_t lines, int64_t k, int64_t kp, const int64_t *__restrict__ eline, int s,
                            int nparts, int8_t *__restrict__ dig, int64_t line, int64_t k0)
{
    const CUtensorMap &mre = *mre_p, &mim = *mim_p;
    extern __shared__ uint8_t tsm_raw[];
    uint8_t *tile = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(tsm_raw) + 1023) & ~uintptr_t(1023));
    constexpr int ROW = 8 * L;                        // bytes per entry row
    constexpr int SWM = L == 16 ? 7 : L == 8 ? 3 : L == 4 ? 1 : 0;   // 16-byte chunk XOR mask
    // digit staging, double-buffered: [2][3 parts][8 planes][kSplitT bytes]
    uint8_t *stage = tile + 2 * kSplitT * ROW;
    uint64_t *bar = reinterpret_cast<uint64_t *>(stage + 2 * 3 * 8 * kSplitT);
    const int tid = threadIdx.x;
    if (tid == 0) { mbar_init(bar, 1); fence_barrier_init(); }
    __syncthreads();
    if (tid == 0) {
        mbar_arrive_expect_tx(bar, 2u * kSplitT * ROW);
        if (side == 0) {                              // dims {L, k, rows}: coords (0, k0, line)
            tma_load_3d(tile, &mre, bar, 0, (int)k0, (int)line);
            tma_load_3d(tile + kSplitT * ROW, &mim, bar, 0, (int)k0, (int)line);
        } else {                                      // dims {L, n, k}: coords (0, line, k0)
            tma_load_3d(tile, &mre, bar, 0, (int)line, (int)k0);
            tma_load_3d(tile + kSplitT * ROW, &mim, bar, 0, (int)line, (int)k0);
        }
    }
    const int64_t kk = k0 + tid;
    const bool valid = kk < k;
    int64_t ex[2] = {0, 0};
    bool neg[2] = {false, false};
    if (valid) {
#pragma unroll
        for (int p = 0; p < 2; p++) {
            const DMat &M = p ? im : re;
            const int64_t idx = side == 0 ? line * M.ld + kk : kk * M.ld + line;
            ex[p] = __ldg(M.exp + idx);
            neg[p] = __ldg(M.sign + idx) != 0;
        }
    }
    const int64_t e = eline[line];
    const int64_t W = 8 * (int64_t)s - 3;
    mbar_wait(bar, 0);
    // limb l of this thread's entry in part p (swizzled shared-memory address)
    // (the swizzle's XOR operand (o >> 7) & SWM is constant per thread: the entry row tid * ROW has
    //  zero low bits wherever the XOR acts)
    const uint32_t xm = (uint32_t)((((tid * ROW) >> 7) & SWM) << 4);
    const uint32_t myrow = smem_u32(tile) + (uint32_t)(tid * ROW);      // shared-space address
    // (limb indices are int32: saturated below at -(nwords + 2) and above at L, which keeps every
    //  word of the walk -- all limbs outside [0, L) read as zero -- with one 32-bit bound check)
    auto limb = [&](int p, int32_t l) -> uint64_t {
        if ((uint32_t)l >= (uint32_t)L) return 0ull;
        uint64_t v;
        asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(myrow + (uint32_t)(p * kSplitT * ROW) + ((uint32_t)(8 * l) ^ xm)));
        return v;
    };
    const int32_t li_lo = -((s + 7) / 8 + 2);
    int32_t li[2]; int bo[2]; uint64_t lo[2], nm[2];
    uint32_t nc[2];                                   // two's complement: x ^ nm + carry (nc starts at neg)
    bool zero[2];
#pragma unroll
    for (int p = 0; p < 2; p++) {
        zero[p] = !valid || limb(p, L - 1) == 0;
        const int64_t pos0 = 64 * (int64_t)L - W + e - ex[p];
        const int64_t l64 = pos0 >= 0 ? (pos0 >> 6) : -((-pos0 + 63) >> 6);
        bo[p] = (int)(pos0 - (l64 << 6));
        li[p] = (int32_t)(l64 < li_lo ? li_lo : l64 > L ? L : l64);
        lo[p] = zero[p] ? 0ull : limb(p, li[p]);
        neg[p] = neg[p] && !zero[p];
        nm[p] = neg[p] ? ~0ull : 0ull;
        nc[p] = neg[p] ? 1u : 0u;
    }
    uint32_t csum = 0, ch[3] = {0, 0, 0};
    const int64_t plane = lines * kp;
    const int64_t rowlen = min((int64_t)kSplitT, kp - k0);          // bytes of this CTA's plane rows
    const int nwords = (s + 7) / 8;
    // full tiles: thread q copies the fixed (part, byte, vector) rows q and q + 128 of the staging
    // every word; their plane rows move down 8 planes per word (a constant pointer step)
    constexpr int VPR = kSplitT / 16;
    int8_t *optr[2]; int ostg[2]; int obt[2]; bool oon[2];
#pragma unroll
    for (int it = 0; it < 2; it++) {
        const int q = tid + it * kSplitT, row = q / VPR, v = q % VPR;
        const int p = row >> 3, bt = row & 7;
        oon[it] = q < nparts * 8 * VPR;
        obt[it] = bt;
        ostg[it] = (p * 8 + bt) * kSplitT + 16 * v;
        optr[it] = dig + ((int64_t)p * s + (s - 1 - bt)) * plane + line * kp + k0 + 16 * v;
    }
    const int64_t ostep = 8 * plane;
    // WS: thread q handles the (part, quad) item q inside this CTA's row length (3 parts x 32 quads
    // <= 128 threads: one item per thread at most)
    constexpr int QIT = (3 * (kSplitT / 4) + kSplitT - 1) / kSplitT;
    static_assert(QIT == 1, "one copy-out item per thread");
    int8_t *qptr[QIT]; int qoff[QIT]; bool qon[QIT];
#pragma unroll
    for (int it = 0; it < QIT; it++) {
        const int q = tid + it * kSplitT, p = q / (kSplitT / 4), c = q % (kSplitT / 4);
        qon[it] = p < nparts && 4 * c < rowlen;
        qoff[it] = (p * kSplitT + 4 * c) * 8;
        qptr[it] = dig + ((int64_t)p * s + (s - 1)) * plane + line * kp + k0 + 4 * c;
    }
    for (int w = 0; w < nwords; w++) {
        uint8_t *stg = stage + (w & 1) * (3 * 8 * kSplitT);
        uint64_t y[3];
#pragma unroll
        for (int p = 0; p < 2; p++) {
            const uint64_t hi = zero[p] ? 0ull : limb(p, li[p] + 1);
            const uint64_t x = funnel64(lo[p], hi, (uint32_t)bo[p]);
            lo[p] = hi; li[p]++;
            y[p] = add64_carry(x ^ nm[p], 0ull, nc[p]);   // negation without a divergent branch
        }
        y[2] = add64_carry(y[0], y[1], csum);         // 3M: Re + Im (two's complement, with carry)
#pragma unroll
        for (int p = 0; p < 3; p++) {                 // + H with carry, XOR 0x80 per byte -> staging
            if (p >= nparts) break;
            const uint64_t d = add64_carry(y[p], kH, ch[p]) ^ kH;
            if constexpr (WS) {                          // [part][entry] words
                asm volatile("st.shared.u64 [%0], %1;" :: "r"(smem_u32(stg) + (uint32_t)((p * kSplitT + tid) * 8)), "l"(d) : "memory");
            } else {
#pragma unroll
                for (int bt = 0; bt < 8; bt++) stg[(p * 8 + bt) * kSplitT + tid] = (uint8_t)(d >> (8 * bt));
            }
        }
        __syncthreads();
        const int nb = min(8, s - 8 * w);
        if constexpr (WS) {
            // item (part p, quad c): the words of entries 4c .. 4c+3; for each of the 8 planes a
            // byte-permute gathers their byte bt into one 32-bit word; a warp's store is one whole
            // 128-byte plane row segment
#pragma unroll
            for (int it = 0; it < QIT; it++) {
                if (!qon[it]) continue;
                uint4 w01, w23;
                const uint32_t qa = smem_u32(stg) + (uint32_t)qoff[it];
                asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(w01.x), "=r"(w01.y), "=r"(w01.z), "=r"(w01.w) : "r"(qa) : "memory");
                asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(w23.x), "=r"(w23.y), "=r"(w23.z), "=r"(w23.w) : "r"(qa + 16) : "memory");
                // 4 x 4 byte transposes (8 permutes per 4 planes): entries e0..e3 = w01.{x,y},
                // w01.{z,w}, w23.{x,y}, w23.{z,w} (low / high 32 bits); plane bt's word is byte bt
                // of e0..e3
                uint32_t pw[8];
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    const uint32_t e0 = h ? w01.y : w01.x, e1 = h ? w01.w : w01.z;
                    const uint32_t e2 = h ? w23.y : w23.x, e3 = h ? w23.w : w23.z;
                    const uint32_t t0 = __byte_perm(e0, e1, 0x5140), t1 = __byte_perm(e2, e3, 0x5140);
                    const uint32_t t2 = __byte_perm(e0, e1, 0x7362), t3 = __byte_perm(e2, e3, 0x7362);
                    pw[4 * h + 0] = __byte_perm(t0, t1, 0x5410);
                    pw[4 * h + 1] = __byte_perm(t0, t1, 0x7632);
                    pw[4 * h + 2] = __byte_perm(t2, t3, 0x5410);
                    pw[4 * h + 3] = __byte_perm(t2, t3, 0x7632);
                }
                int8_t *o = qptr[it];
                if (nb == 8) {
#pragma unroll
                    for (int bt = 0; bt < 8; bt++, o -= plane) *reinterpret_cast<uint32_t *>(o) = pw[bt];
                } else {
#pragma unroll
                    for (int bt = 0; bt < 8; bt++, o -= plane)
                        if (bt < nb) *reinterpret_cast<uint32_t *>(o) = pw[bt];
                }
                qptr[it] -= ostep;
            }
            continue;
        }
        // plane rows of this word: (part p, byte bt) -> plane s-1-(8w+bt), 16-byte vector stores
        if (rowlen == kSplitT) {                       // full tile: 8 vectors per row, no divisions
#pragma unroll
            for (int it = 0; it < 2; it++) {
                if (oon[it] && obt[it] < nb)
                    *reinterpret_cast<uint4 *>(optr[it]) = *reinterpret_cast<const uint4 *>(stg + ostg[it]);
                optr[it] -= ostep;
            }
            continue;
        }
        const int vec_per_row = (int)((rowlen + 15) / 16);
        for (int q = tid; q < nparts * 8 * vec_per_row; q += kSplitT) {
            const int row = q / vec_per_row, v = q - row * vec_per_row;
            const int p = row >> 3, bt = row & 7;
            if (bt >= nb) continue;
            int8_t *o = dig + ((int64_t)p * s + (s - 1 - 8 * w - bt)) * plane + line * kp + k0 + 16 * v;
            const uint4 val = *reinterpret_cast<const uint4 *>(stg + (p * 8 + bt) * kSplitT + 16 * v);
            if (16 * v + 16 <= rowlen) *reinterpret_cast<uint4 *>(o) = val;
            else {
                const uint8_t *vb = reinterpret_cast<const uint8_t *>(&val);
                for (int x = 0; 16 * v + x < rowlen; x++) o[x] = (int8_t)vb[x];
            }
        }
        // (the other staging buffer is written next; the one stored here is rewritten only after
        //  the next word's __syncthreads)
    }
}

template <int L, bool WS = true>
__global__ void __launch_bounds__(kSplitT)
split_tma_kernel(const __grid_constant__ CUtensorMap mre, const __grid_constant__ CUtensorMap mim, DMat re, DMat im,
                 int side, int64_t lines, int64_t k, int64_t kp, const int64_t *__restrict__ eline, int s, int nparts,
                 int8_t *__restrict__ dig, const DevRuleState *drs)
{
    if (drs) { if (drs->status) return; s = drs->cur.s; }    // device rule: the chosen s
    split_tma_body<L, WS>(&mre, &mim, re, im, side, lines, k, kp, eline, s, nparts, dig, blockIdx.y,
                          (int64_t)blockIdx.x * kSplitT);
}

// both operands in one launch: block rows [0, n) split the columns of B, [n, n + m) the rows of A
template <int L>
__global__ void __launch_bounds__(kSplitT)
split2_tma_kernel(const __grid_constant__ CUtensorMap mAre, const __grid_constant__ CUtensorMap mAim,
                  const __grid_constant__ CUtensorMap mBre, const __grid_constant__ CUtensorMap mBim, DMat Are, DMat Aim,
                  DMat Bre, DMat Bim, int64_t m, int64_t n, int64_t k, int64_t kp, const int64_t *__restrict__ eA,
                  const int64_t *__restrict__ eB, int s, int nparts, int8_t *__restrict__ digA, int8_t *__restrict__ digB,
                  const DevRuleState *drs)
{
    pdl_wait();
    if (drs) { if (drs->status) return; s = drs->cur.s; }
    const int64_t y = blockIdx.y, k0 = (int64_t)blockIdx.x * kSplitT;
    if (y < n) split_tma_body<L, true>(&mBre, &mBim, Bre, Bim, 1, n, k, kp, eB, s, nparts, digB, y, k0);
    else       split_tma_body<L, true>(&mAre, &mAim, Are, Aim, 0, m, k, kp, eA, s, nparts, digA, y - n, k0);
}

template <int L>
static cudaError_t split_tma_launch_t(DMat re, DMat im, int side, int64_t lines, int64_t k, int64_t kp,
                                      const int64_t *eline, int s, int nparts, int8_t *dig, const DevRuleState *drs,
                                      cudaStream_t st)
{
    static const bool bytestg = getenv("MPCGEMM_SPLIT_BYTESTG") != nullptr;   // round-1 byte staging
    alignas(64) uint8_t mre[128], mim[128];           // CUtensorMap storage
    for (int p = 0; p < 2; p++) {
        const DMat &M = p ? im : re;
        int rc;
        if (side == 0)      // A (lines x k): dims {L, k, lines}
            rc = encode_limb_map(p ? mim : mre, M.limbs, L, (uint64_t)k, (uint64_t)lines, 8ull * L, 8ull * L * M.ld, kSplitT, 1);
        else                // B (k x lines): dims {L, lines, k}
            rc = encode_limb_map(p ? mim : mre, M.limbs, L, (uint64_t)lines, (uint64_t)k, 8ull * L, 8ull * L * M.ld, 1, kSplitT);
        if (rc) return cudaErrorInvalidValue;
    }
    const size_t sm = 1024 + 2 * (size_t)kSplitT * 8 * L + 2 * 3 * 8 * kSplitT + 64;
    auto kern = bytestg ? split_tma_kernel<L, false> : split_tma_kernel<L, true>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    dim3 grid((unsigned)((kp + kSplitT - 1) / kSplitT), (unsigned)lines);
    kern<<<grid, kSplitT, sm, st>>>(*reinterpret_cast<const CUtensorMap *>(mre), *reinterpret_cast<const CUtensorMap *>(mim),
                                    re, im, side, lines, k, kp, eline, s, nparts, dig, drs);
    return cudaGetLastError();
}

template <int L>
static cudaError_t split2_launch_t(DMat Are, DMat Aim, DMat Bre, DMat Bim, int64_t m, int64_t n, int64_t k, int64_t kp,
                                   const int64_t *eA, const int64_t *eB, int s, int nparts, int8_t *digA, int8_t *digB,
                                   const DevRuleState *drs, cudaStream_t st)
{
    alignas(64) uint8_t maps[4][128];                 // A re, A im, B re, B im
    const DMat *M[4] = {&Are, &Aim, &Bre, &Bim};
    for (int q = 0; q < 4; q++) {
        const int rc = q < 2 ? encode_limb_map(maps[q], M[q]->limbs, L, (uint64_t)k, (uint64_t)m, 8ull * L, 8ull * L * M[q]->ld, kSplitT, 1)
                             : encode_limb_map(maps[q], M[q]->limbs, L, (uint64_t)n, (uint64_t)k, 8ull * L, 8ull * L * M[q]->ld, 1, kSplitT);
        if (rc) return cudaErrorInvalidValue;
    }
    const size_t sm = 1024 + 2 * (size_t)kSplitT * 8 * L + 2 * 3 * 8 * kSplitT + 64;
    cudaError_t e = cudaFuncSetAttribute(split2_tma_kernel<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    dim3 grid((unsigned)((kp + kSplitT - 1) / kSplitT), (unsigned)(m + n));
    auto cm = [&](int q) { return *reinterpret_cast<const CUtensorMap *>(maps[q]); };
    return launch_pdl(split2_tma_kernel<L>, grid, dim3(kSplitT), sm, st, cm(0), cm(1), cm(2), cm(3), Are, Aim, Bre, Bim, m, n,
                      k, kp, eA, eB, s, nparts, digA, digB, drs);
}

// a-3 for B and A in one launch when the TMA path applies (else two split_launch calls)
cudaError_t split2_launch(DMat Are, DMat Aim, DMat Bre, DMat Bim, int64_t m, int64_t n, int64_t k, int64_t kp, int L,
                          const int64_t *eA, const int64_t *eB, int s, int nparts, int8_t *digA, int8_t *digB,
                          cudaStream_t st, const DevRuleState *drs, int *nlaunch)
{
    if (nlaunch) *nlaunch = 1;
    const bool aligned = !(reinterpret_cast<uintptr_t>(Are.limbs) & 15) && !(reinterpret_cast<uintptr_t>(Aim.limbs) & 15) &&
                         !(reinterpret_cast<uintptr_t>(Bre.limbs) & 15) && !(reinterpret_cast<uintptr_t>(Bim.limbs) & 15);
    if (m > 0 && n > 0 && kp > 0 && m + n < 65536 && aligned && !getenv("MPCGEMM_SPLIT_V1") &&
        !getenv("MPCGEMM_SPLIT_BYTESTG")) {
        cudaError_t e = cudaErrorNotSupported;
        switch (L) {
            case 16: e = split2_launch_t<16>(Are, Aim, Bre, Bim, m, n, k, kp, eA, eB, s, nparts, digA, digB, drs, st); break;
            case 14: e = split2_launch_t<14>(Are, Aim, Bre, Bim, m, n, k, kp, eA, eB, s, nparts, digA, digB, drs, st); break;
            case 12: e = split2_launch_t<12>(Are, Aim, Bre, Bim, m, n, k, kp, eA, eB, s, nparts, digA, digB, drs, st); break;
            case 10: e = split2_launch_t<10>(Are, Aim, Bre, Bim, m, n, k, kp, eA, eB, s, nparts, digA, digB, drs, st); break;
            case 8:  e = split2_launch_t<8>(Are, Aim, Bre, Bim, m, n, k, kp, eA, eB, s, nparts, digA, digB, drs, st); break;
            case 6:  e = split2_launch_t<6>(Are, Aim, Bre, Bim, m, n, k, kp, eA, eB, s, nparts, digA, digB, drs, st); break;
            case 4:  e = split2_launch_t<4>(Are, Aim, Bre, Bim, m, n, k, kp, eA, eB, s, nparts, digA, digB, drs, st); break;
            case 2:  e = split2_launch_t<2>(Are, Aim, Bre, Bim, m, n, k, kp, eA, eB, s, nparts, digA, digB, drs, st); break;
            default: break;
        }
        if (e != cudaErrorNotSupported && e != cudaErrorInvalidValue) return e;
    }
    if (nlaunch) *nlaunch = 2;
    cudaError_t e = split_launch(Bre, Bim, 1, n, k, kp, L, eB, s, nparts, digB, st, drs);
    if (e != cudaSuccess) return e;
    return split_launch(Are, Aim, 0, m, k, kp, L, eA, s, nparts, digA, st, drs);
}

cudaError_t split_launch(DMat re, DMat im, int side, int64_t lines, int64_t k, int64_t kp, int L,
                         const int64_t *eline, int s, int nparts, int8_t *dig, cudaStream_t st, const DevRuleState *drs)
{
    if (lines == 0 || kp == 0) return cudaSuccess;
    const bool tma_ok = lines < 65536 && getenv("MPCGEMM_SPLIT_V1") == nullptr &&
                        !(reinterpret_cast<uintptr_t>(re.limbs) & 15) && !(reinterpret_cast<uintptr_t>(im.limbs) & 15);
    if (tma_ok) {
        cudaError_t e = cudaErrorNotSupported;
        if (L == 16) e = split_tma_launch_t<16>(re, im, side, lines, k, kp, eline, s, nparts, dig, drs, st);
        else if (L == 8) e = split_tma_launch_t<8>(re, im, side, lines, k, kp, eline, s, nparts, dig, drs, st);
        else if (L == 4) e = split_tma_launch_t<4>(re, im, side, lines, k, kp, eline, s, nparts, dig, drs, st);
        else if (L == 2) e = split_tma_launch_t<2>(re, im, side, lines, k, kp, eline, s, nparts, dig, drs, st);
        // other even L: unswizzled tiles (8L-byte rows; the bank conflicts of the per-entry limb
        // reads cost far less than the per-thread-streams kernel's L2 re-fetches)
        else if (L == 12) e = split_tma_launch_t<12>(re, im, side, lines, k, kp, eline, s, nparts, dig, drs, st);
        else if (L == 6) e = split_tma_launch_t<6>(re, im, side, lines, k, kp, eline, s, nparts, dig, drs, st);
        else if (L == 10) e = split_tma_launch_t<10>(re, im, side, lines, k, kp, eline, s, nparts, dig, drs, st);
        else if (L == 14) e = split_tma_launch_t<14>(re, im, side, lines, k, kp, eline, s, nparts, dig, drs, st);
        if (e != cudaErrorNotSupported && e != cudaErrorInvalidValue) return e;
    }
    const int64_t threads = (kp + kSplitVec - 1) / kSplitVec;
    dim3 grid((unsigned)((threads + 127) / 128), (unsigned)(lines < 65535 ? lines : 65535));
    split_kernel<<<grid, 128, 0, st>>>(re, im, side, lines, k, kp, L, eline, s, nparts, dig, drs);
    return cudaGetLastError();
}

// ================================================================== a-2: pre-pass
// relative entry exponents for the max-plus stage: real entries clamped to [-2^28, 0], zero
// entries -2^30, so a sum is > -2^30 iff both entries are nonzero (no int32 overflow:
// sentinel + sentinel = -2^31)
constexpr int32_t kRelSentinel = -(1 << 30);
constexpr int32_t kRelClamp = -(1 << 28);

// one pre-pass plane entry (line, kk < k) of a side: t = the top 7 bits of the larger part below
// the line's exponent e, rel = the entry's exponent relative to e (clamped; sentinel if zero)
MPC_DEV void planes_entry(const DMat &re, const DMat &im, int side, int64_t line, int64_t kk, int L, int64_t e,
                          int &best, int32_t &r)
{
    best = 0;
    int64_t emax = 0; bool any = false;
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
    r = kRelSentinel;
    if (any) {
        int64_t d = emax - e;                          // <= 0
        r = d < kRelClamp ? kRelClamp : (int32_t)d;
    }
}

// the same entry from the a-1 scan's top bytes b0, b1 (Re, Im; linemax_body) and the exponents
MPC_DEV void planes_entry_tb(const DMat &re, const DMat &im, int side, int64_t line, int64_t kk, int64_t e, uint8_t b0,
                             uint8_t b1, int &best, int32_t &r)
{
    best = 0;
    int64_t emax = 0; bool any = false;
#pragma unroll
    for (int p = 0; p < 2; p++) {
        const uint8_t b = p ? b1 : b0;
        if (!b) continue;
        const DMat &M = p ? im : re;
        const int64_t ex = __ldg(M.exp + (side == 0 ? line * M.ld + kk : kk * M.ld + line));
        const int64_t d = e - ex;                      // >= 0; t = top >> (57 + d) for d <= 6, else 0
        const int tv = d <= 6 ? (int)(b >> (1 + d)) : 0;
        best = tv > best ? tv : best;
        if (!any || ex > emax) emax = ex;
        any = true;
    }
    r = kRelSentinel;
    if (any) {
        const int64_t dd = emax - e;
        r = dd < kRelClamp ? kRelClamp : (int32_t)dd;
    }
}

MPC_DEV void prepass_planes_body(const DMat &re, const DMat &im, int side, int64_t lines, int64_t k, int64_t kp, int L,
                                 const int64_t *__restrict__ eline, int8_t *t, int32_t *rel, int64_t bx, int64_t by,
                                 int64_t gy, const uint8_t *tb = nullptr, int64_t tbpart = 0)
{
    const int64_t kk = bx * blockDim.x + threadIdx.x;
    if (kk >= kp) return;
    for (int64_t line = by; line < lines; line += gy) {
        int best = 0;
        int32_t r = kRelSentinel;
        if (kk < k) {
            if (tb) planes_entry_tb(re, im, side, line, kk, eline[line], tb[line * kp + kk], tb[tbpart + line * kp + kk], best, r);
            else planes_entry(re, im, side, line, kk, L, eline[line], best, r);
        }
        t[line * kp + kk] = (int8_t)best;
        rel[line * kp + kk] = r;
    }
}

__global__ void prepass_planes_kernel(DMat re, DMat im, int side, int64_t lines, int64_t k, int64_t kp, int L,
                                      const int64_t *__restrict__ eline, int8_t *t, int32_t *rel)
{
    prepass_planes_body(re, im, side, lines, k, kp, L, eline, t, rel, blockIdx.x, blockIdx.y, gridDim.y);
}

__global__ void prepass_planes2_kernel(DMat re0, DMat im0, int64_t lines0, const int64_t *eline0, int8_t *t0, int32_t *rel0,
                                       DMat re1, DMat im1, int64_t lines1, const int64_t *eline1, int8_t *t1, int32_t *rel1,
                                       int64_t k, int64_t kp, int L, int64_t gx, int64_t gy0, int64_t gy1,
                                       unsigned long long *fill0, int64_t nfill0, unsigned long long *fill1, int64_t nfill1,
                                       const uint8_t *tb)
{
    pdl_wait();
    const int64_t b = blockIdx.x;
    if (b == 0) {                                      // the stage-1/2 reduction targets: all ones
        for (int64_t i = threadIdx.x; i < nfill0; i += blockDim.x) fill0[i] = ~0ull;   // (replaces two
        for (int64_t i = threadIdx.x; i < nfill1; i += blockDim.x) fill1[i] = ~0ull;   //  memset nodes)
    }
    // (tb: [part][A rows then B columns][kp] top bytes from the a-1 scan, or null)
    const int64_t tbpart = (lines0 + lines1) * kp;
    if (b < gx * gy0)
        prepass_planes_body(re0, im0, 0, lines0, k, kp, L, eline0, t0, rel0, b % gx, b / gx, gy0, tb, tbpart);
    else {
        const int64_t c = b - gx * gy0;
        prepass_planes_body(re1, im1, 1, lines1, k, kp, L, eline1, t1, rel1, c % gx, c / gx, gy1,
                            tb ? tb + lines0 * kp : nullptr, tbpart);
    }
}

cudaError_t prepass_planes2_launch(DMat Are, DMat Aim, DMat Bre, DMat Bim, int64_t m, int64_t n, int64_t k, int64_t kp,
                                   int L, const int64_t *eA, const int64_t *eB, int8_t *tA, int32_t *relA, int8_t *tB,
                                   int32_t *relB, cudaStream_t st, unsigned long long *fill0, int64_t nfill0,
                                   unsigned long long *fill1, int64_t nfill1, const uint8_t *tb)
{
    if (kp == 0 || m + n == 0) {
        cudaError_t e = nfill0 ? cudaMemsetAsync(fill0, 0xFF, 8 * nfill0, st) : cudaSuccess;
        if (e == cudaSuccess && nfill1) e = cudaMemsetAsync(fill1, 0xFF, 8 * nfill1, st);
        return e;
    }
    const int64_t gx = (kp + 127) / 128, gy0 = std::min<int64_t>(m, 32768), gy1 = std::min<int64_t>(n, 32768);
    return launch_pdl(prepass_planes2_kernel, dim3((unsigned)(gx * (gy0 + gy1))), dim3(128), 0, st, Are, Aim, m, eA, tA,
                      relA, Bre, Bim, n, eB, tB, relB, k, kp, L, gx, gy0, gy1, fill0, nfill0, fill1, nfill1, tb);
}

cudaError_t prepass_planes_launch(DMat re, DMat im, int side, int64_t lines, int64_t k, int64_t kp, int L,
                                  const int64_t *eline, int8_t *t, int32_t *rel, cudaStream_t st)
{
    if (lines == 0 || kp == 0) return cudaSuccess;
    dim3 grid((unsigned)((kp + 127) / 128), (unsigned)(lines < 65535 ? lines : 65535));
    prepass_planes_kernel<<<grid, 128, 0, st>>>(re, im, side, lines, k, kp, L, eline, t, rel);
    return cudaGetLastError();
}

MPC_DEV int64_t sum_T(const int32_t *T, int nslots, int64_t nstrips, int64_t i, int64_t j) {
    int64_t v = 0;
    for (int q = 0; q < nslots; q++) v += T[part_off(i, j, q, nslots, nstrips)];
    return v;
}

// stage 1: min over nonzero line pairs of T_ij, per 256-row block (out_min[i >> 8]; the
// global value is the min over blocks, NEXT-4 uses each block's own).  Each CTA takes one
// contiguous range of (i, j) -- a few rows, so (nearly) one 256-row block -- keeps a running
// minimum per thread, and reduces over the warp and the CTA before ONE atomic per row block it
// touched (a global atomic per warp on the ~m/256 targets serialised in L2: 82-91 us at configs
// 4 and 5 before)
__global__ void __launch_bounds__(256)
prepass_min_kernel(const int32_t *T, int nslots, int64_t nstrips, int64_t m, int64_t n,
                   const uint8_t *nzA, const uint8_t *nzB, unsigned long long *out_min)
{
    __shared__ unsigned long long wv[8];
    __shared__ long long wb[8];
    const int64_t total = m * n;
    const int64_t per = (total + gridDim.x - 1) / gridDim.x;
    const int64_t beg = (int64_t)blockIdx.x * per, end = min(total, beg + per);
    unsigned long long v = ULLONG_MAX;
    int64_t vb = -1;                                  // the row block v belongs to
    int64_t i = (beg + threadIdx.x) / n, j = beg + threadIdx.x - i * n;   // one division; then stepped
    for (int64_t t = beg + threadIdx.x; t < end; t += blockDim.x, j += blockDim.x) {
        while (j >= n) { j -= n; i++; }
        const int64_t b = i >> kSBlkShift;
        if (b != vb) {                                // (at most once per row-block boundary)
            if (vb >= 0 && v != ULLONG_MAX) atomicMin(out_min + vb, v);
            v = ULLONG_MAX; vb = b;
        }
        if (nzA[i] && nzB[j]) {
            const unsigned long long x = (unsigned long long)sum_T(T, nslots, nstrips, i, j);
            v = x < v ? x : v;
        }
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long b0 = __shfl_sync(0xffffffffu, vb, 0);
    if (__all_sync(0xffffffffu, vb == b0 || vb < 0)) {
#pragma unroll
        for (int o = 16; o; o >>= 1) { const unsigned long long y = __shfl_xor_sync(0xffffffffu, v, o); v = y < v ? y : v; }
        if (lane == 0) { wv[warp] = v; wb[warp] = b0; }
    } else {
        if (vb >= 0 && v != ULLONG_MAX) atomicMin(out_min + vb, v);
        if (lane == 0) { wv[warp] = ULLONG_MAX; wb[warp] = -1; }
    }
    __syncthreads();
    if (threadIdx.x == 0) {                           // merge the warps; one atomic per row block
        unsigned long long cv = ULLONG_MAX;
        long long cb = -1;
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) {
            if (wb[w] < 0 || wv[w] == ULLONG_MAX) continue;
            if (wb[w] != cb) {
                if (cb >= 0) atomicMin(out_min + cb, cv);
                cb = wb[w]; cv = wv[w];
            } else cv = wv[w] < cv ? wv[w] : cv;
        }
        if (cb >= 0) atomicMin(out_min + cb, cv);
    }
}

// stage 2: exact max-plus exponent bound and the per-pair bound choice
MPC_DEV void maxplus_body(const int32_t *T, int nslots, int64_t nstrips, int64_t m, int64_t n,
                          int64_t k, int64_t kp, const uint8_t *nzA, const uint8_t *nzB,
                          const int32_t *relA, const int32_t *relB,
                          unsigned long long *out_min, unsigned long long *out_min1, long long *out_max2,
                          const unsigned long long *gate, int64_t ngate, int64_t i0, int64_t j0)
{
    __shared__ int32_t sa[32][33], sb[32][33];
    if (gate) {                                       // device rule: run only if a block's stage-1 min is 0
        int z = 0;
        for (int64_t b = threadIdx.x; b < ngate; b += blockDim.x) z |= __ldcg(gate + b) == 0;
        if (!__syncthreads_or(z)) return;
    }
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;    // 32 x 8 (tile origin i0, j0)
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
        const int64_t Tv = sum_T(T, nslots, nstrips, i, j);
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
    if (tx == 0) {                                    // a 32-row tile lies in one 256-row block
        const int64_t b = i0 >> kSBlkShift;
        if (lmin != ULLONG_MAX) atomicMin(out_min + b, lmin);
        if (lmin1 != ULLONG_MAX) atomicMin(out_min1 + b, lmin1);
        if (lmax2 >= 0) atomicMax(out_max2 + b, lmax2);
    }
}

__global__ void __launch_bounds__(256)
prepass_maxplus_kernel(const int32_t *T, int nslots, int64_t nstrips, int64_t m, int64_t n,
                       int64_t k, int64_t kp, const uint8_t *nzA, const uint8_t *nzB,
                       const int32_t *relA, const int32_t *relB,
                       unsigned long long *out_min, unsigned long long *out_min1, long long *out_max2,
                       const unsigned long long *gate = nullptr, int64_t ngate = 0)
{
    maxplus_body(T, nslots, nstrips, m, n, k, kp, nzA, nzB, relA, relB, out_min, out_min1, out_max2, gate, ngate,
                 (int64_t)blockIdx.y * 32, (int64_t)blockIdx.x * 32);
}

__global__ void readback_kernel(uint32_t *dst, const uint32_t *src, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

cudaError_t readback_launch(void *dst_mapped, const void *src, size_t bytes, cudaStream_t st) {
    const int64_t n = (int64_t)(bytes / 4);            // callers pass multiples of 4 bytes
    if (n == 0) return cudaSuccess;
    readback_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 64), 256, 0, st>>>((uint32_t *)dst_mapped,
                                                                                      (const uint32_t *)src, n);
    return cudaGetLastError();
}

// device rule: the host path's reduction over 256-row blocks and slice rule (mpcgemm.cu
// run_prepass / gemm_impl; rule.cuh), one warp (threads 0..31 of the calling block); picks the
// candidate plan of the certified s
MPC_DEV void rule_body(const unsigned long long *min1, const unsigned long long *min2,
                       const unsigned long long *min12, const long long *max22, int64_t nb, int64_t k, int prec,
                       int method, const DevPlan *plans, int s_lo, int s_hi, DevRuleState *drs, double *lr_shp)
{
    // lanes test 32 consecutive candidate s at a time from s_lo - 1 on, with rule_slices' predicate
    // (the rule at log2 rho-hat >= 0 cannot pick below s_lo), then lane 0 finishes
    double &lr_sh = *lr_shp;
    if (threadIdx.x == 0) {
    bool any0 = false;
    for (int64_t b = 0; b < nb; b++) any0 = any0 || min1[b] == 0;
    int64_t g0 = -1, g1 = -1, g2 = -1;
    for (int64_t b = 0; b < nb; b++) {
        int64_t t0, t1, t2;
        if (!any0) { t0 = min1[b] == ULLONG_MAX ? -1 : (int64_t)min1[b]; t1 = t0; t2 = -1; }
        else {
            t0 = min2[b] == ULLONG_MAX ? -1 : (int64_t)min2[b];
            t1 = min12[b] == ULLONG_MAX ? -1 : (int64_t)min12[b];
            t2 = (int64_t)max22[b];
        }
        if (t0 >= 0 && (g0 < 0 || t0 < g0)) g0 = t0;
        if (t1 >= 0 && (g1 < 0 || t1 < g1)) g1 = t1;
        if (t2 > g2) g2 = t2;
    }
    if (g0 < 0) { g1 = g2 = -1; }
    else if (g0 > 0) { g1 = g0; g2 = -1; }
    lr_sh = rule_log2rho(k, g0, g1, g2);
    drs->minT = g0; drs->minT1 = g1; drs->maxD2 = g2;
    }
    __syncwarp();
    const double lr = lr_sh;
    const double c = method == 3 ? 4.0 : 3.0;
    int sv = -8;
    for (int base = max(1, s_lo - 1); base <= kMaxSlices; base += 32) {
        const int cand = base + (int)threadIdx.x;
        const bool ok = cand <= kMaxSlices && 8.0 * cand >= (double)prec - 4.0 + log2(c * cand) + lr + 0.1;
        const unsigned bal = __ballot_sync(0xffffffffu, ok);
        if (bal) { sv = base + __ffs(bal) - 1; break; }
    }
    if (threadIdx.x) return;
    drs->s_needed = sv;
    if (sv >= s_lo && sv <= s_hi) { drs->cur = plans[sv - s_lo]; drs->status = 0; }
    else { drs->cur = DevPlan{nullptr, nullptr, nullptr, sv, 0, 0, 0}; drs->status = -8; }
}

__global__ void rule_kernel(const unsigned long long *min1, const unsigned long long *min2,
                            const unsigned long long *min12, const long long *max22, int64_t nb, int64_t k, int prec,
                            int method, const DevPlan *plans, int s_lo, int s_hi, DevRuleState *drs)
{
    __shared__ double lr_sh;
    if (blockIdx.x) return;
    rule_body(min1, min2, min12, max22, nb, k, prec, method, plans, s_lo, s_hi, drs, &lr_sh);
}

// stage 2 (gated) + the rule in one launch: every block counts itself done on a counter that the
// caller's all-ones memset of the stage-2 arrays initialised to 0xFFFFFFFF, and the last block's
// first warp runs the rule (no launch of its own)
__global__ void __launch_bounds__(256)
prepass_maxplus_rule_kernel(const int32_t *T, int nslots, int64_t nstrips, int64_t m, int64_t n, int64_t k, int64_t kp,
                            const uint8_t *nzA, const uint8_t *nzB, const int32_t *relA, const int32_t *relB,
                            const unsigned long long *min1, unsigned long long *min2, unsigned long long *min12,
                            long long *max22, int64_t nb, int prec, int method, const DevPlan *plans, int s_lo, int s_hi,
                            DevRuleState *drs, unsigned int *done)
{
    pdl_wait();
    maxplus_body(T, nslots, nstrips, m, n, k, kp, nzA, nzB, relA, relB, min2, min12, max22, min1, nb,
                 (int64_t)blockIdx.y * 32, (int64_t)blockIdx.x * 32);
    __shared__ int last;
    __shared__ double lr_sh;
    __syncthreads();
    const unsigned int total = gridDim.x * gridDim.y;
    if (threadIdx.x == 0) { __threadfence(); last = atomicAdd(done, 1u) == total - 2u; }   // from 0xFFFFFFFF
    __syncthreads();
    if (!last || threadIdx.x >= 32) return;
    __threadfence();
    rule_body(min1, min2, min12, max22, nb, k, prec, method, plans, s_lo, s_hi, drs, &lr_sh);
}

// Small shapes (device rule, m n k <= 2^27): T and the stage-1 minimum in ONE launch, without the
// tcgen05 T GEMM.  Each 32 x 32 output tile computes T_ij = sum_k t_ik u_jk itself with dp4a on the
// planes' bytes (the t / u digits are in [0, 127] and zero beyond k, so the int32 sum is the s = 1
// slice GEMM's exact T for k <= 65536), stores it as ONE partial plane (part_off layout, nslots = 1)
// for the gated stage 2, and adds the tile's minimum over nonzero line pairs to its 256-row block.
// Replaces the T GEMM and the stage-1 min kernel (two launches).
MPC_DEV void small_t_tile(const int8_t *tA, const int8_t *tB, int64_t m, int64_t n, int64_t kp, const uint8_t *nzA,
                          const uint8_t *nzB, int32_t *T, int64_t nstrips, unsigned long long *min1, int64_t i0, int64_t j0)
{
    __shared__ uint32_t ta[32][33], tb[32][33];       // 128 k of t / u per row as 32 words
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;    // 32 x 8
    int32_t tv[4] = {0, 0, 0, 0};
    for (int64_t k0 = 0; k0 < kp; k0 += 128) {
        __syncthreads();
        for (int q = threadIdx.x; q < 32 * 32; q += 256) {   // (kp is a multiple of 16: a word is
            const int rr = q >> 5, w = q & 31;               //  inside the row or past its end)
            const int64_t kk = k0 + 4 * w;
            ta[rr][w] = (i0 + rr < m && kk < kp) ? *reinterpret_cast<const uint32_t *>(tA + (i0 + rr) * kp + kk) : 0u;
            tb[rr][w] = (j0 + rr < n && kk < kp) ? *reinterpret_cast<const uint32_t *>(tB + (j0 + rr) * kp + kk) : 0u;
        }
        __syncthreads();
#pragma unroll
        for (int e = 0; e < 4; e++) {
            int32_t acc = tv[e];
            const int r_ = ty * 4 + e;
#pragma unroll 8
            for (int w = 0; w < 32; w++) acc = __dp4a((int)ta[r_][w], (int)tb[tx][w], acc);   // bytes in [0, 127]
            tv[e] = acc;
        }
    }
    unsigned long long l1 = ULLONG_MAX;
    for (int e = 0; e < 4; e++) {
        const int64_t i = i0 + ty * 4 + e, j = j0 + tx;
        if (i >= m || j >= n) continue;
        T[part_off(i, j, 0, 1, nstrips)] = tv[e];
        if (nzA[i] && nzB[j]) l1 = (unsigned long long)tv[e] < l1 ? (unsigned long long)tv[e] : l1;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const unsigned long long y = __shfl_xor_sync(0xffffffffu, l1, o);
        l1 = y < l1 ? y : l1;
    }
    if (tx == 0 && l1 != ULLONG_MAX) atomicMin(min1 + (i0 >> kSBlkShift), l1);   // one 256-row block
}

__global__ void __launch_bounds__(256)
prepass_small_t_kernel(const int8_t *tA, const int8_t *tB, int64_t m, int64_t n, int64_t k, int64_t kp,
                       const uint8_t *nzA, const uint8_t *nzB, int32_t *T, int64_t nstrips, unsigned long long *min1)
{
    pdl_wait();
    small_t_tile(tA, tB, m, n, kp, nzA, nzB, T, nstrips, min1, (int64_t)blockIdx.y * 32, (int64_t)blockIdx.x * 32);
}

cudaError_t prepass_small_t_launch(const int8_t *tA, const int8_t *tB, int64_t m, int64_t n, int64_t k, int64_t kp,
                                   const uint8_t *nzA, const uint8_t *nzB, int32_t *T, int64_t nstrips,
                                   unsigned long long *min1, cudaStream_t st)
{
    if (m <= 0 || n <= 0 || k > 65536) return cudaErrorInvalidValue;
    dim3 grid((unsigned)((n + 31) / 32), (unsigned)((m + 31) / 32));
    return launch_pdl(prepass_small_t_kernel, grid, dim3(256), 0, st, tA, tB, m, n, k, kp, nzA, nzB, T, nstrips, min1);
}

cudaError_t prepass_rule_launch(const int32_t *T, int nslots, int64_t nstrips, int64_t m, int64_t n, int64_t k,
                                int64_t kp, const uint8_t *nzA, const uint8_t *nzB, const int32_t *relA,
                                const int32_t *relB, const unsigned long long *min1, unsigned long long *min2,
                                unsigned long long *min12, long long *max22, int prec, int method,
                                const DevPlan *plans, int s_lo, int s_hi, DevRuleState *drs, cudaStream_t st)
{
    const int64_t nb = (m + kSBlk - 1) / kSBlk;
    if (m > 0 && n > 0 && !getenv("MPCGEMM_RULE_SEPARATE")) {
        // the done counter follows max22[nb] (covered by the caller's all-ones memset)
        unsigned int *done = reinterpret_cast<unsigned int *>(max22 + nb);
        dim3 grid((unsigned)((n + 31) / 32), (unsigned)((m + 31) / 32));
        return launch_pdl(prepass_maxplus_rule_kernel, grid, dim3(256), 0, st, T, nslots, nstrips, m, n, k, kp, nzA, nzB,
                          relA, relB, min1, min2, min12, max22, nb, prec, method, plans, s_lo, s_hi, drs, done);
    }
    if (m > 0 && n > 0) {
        dim3 grid((unsigned)((n + 31) / 32), (unsigned)((m + 31) / 32));
        prepass_maxplus_kernel<<<grid, 256, 0, st>>>(T, nslots, nstrips, m, n, k, kp, nzA, nzB, relA, relB,
                                                     min2, min12, max22, min1, nb);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    rule_kernel<<<1, 32, 0, st>>>(min1, min2, min12, max22, nb, k, prec, method, plans, s_lo, s_hi, drs);
    return cudaGetLastError();
}

cudaError_t prepass_reduce_launch(const int32_t *T, int nslots, int64_t nstrips,
                                  int64_t m, int64_t n, int64_t k, int64_t kp,
                                  const uint8_t *nzA, const uint8_t *nzB, const int32_t *relA, const int32_t *relB,
                                  int stage, unsigned long long *out_min, unsigned long long *out_min1,
                                  long long *out_max2, cudaStream_t st)
{
    if (m == 0 || n == 0) return cudaSuccess;
    if (stage == 1) {
        int64_t blocks = (m * n + 255) / 256;
        if (blocks > 148 * 16) blocks = 148 * 16;
        prepass_min_kernel<<<(unsigned)blocks, 256, 0, st>>>(T, nslots, nstrips, m, n, nzA, nzB, out_min);
    } else {
        dim3 grid((unsigned)((n + 31) / 32), (unsigned)((m + 31) / 32));
        prepass_maxplus_kernel<<<grid, 256, 0, st>>>(T, nslots, nstrips, m, n, k, kp, nzA, nzB, relA, relB,
                                                     out_min, out_min1, out_max2);
    }
    return cudaGetLastError();
}

// ================================================================== a-5 + a-6: fold and normalize
// One thread per output element (i, j); a block covers FOLD_T consecutive j of one row.
// The two's complement fixed-point accumulator of each part lives in shared memory as
// fix[part][limb][thread] (column per thread: conflict-free), built bottom-up:
//     carry += D_r ; emit byte (carry & 0xFF) ; carry >>= 8        r = s+1 .. 2
// with D_r the Eq. 5 / Eq. 6 combination of the job partials (sum of their chunks), then the
// final carry sign-extended at bit 8s.  normalize_store rounds it once (RNE) to prec bits.
struct FixView {
    const uint64_t *base;   // fix[0][thread]
    int64_t stride;         // distance between consecutive limbs
    int n;                  // limbs
    MPC_DEV uint64_t at(int64_t l) const { return (l >= 0 && l < n) ? base[l * stride] : 0ull; }
    MPC_DEV uint64_t bits64(int64_t pos) const {
        if (pos <= -64) return 0;
        if (pos < 0) return at(0) << (-pos);
        const int64_t li = pos >> 6;
        const int bo = (int)(pos & 63);
        const uint64_t lo = at(li);
        if (!bo) return lo;
        return (lo >> bo) | (at(li + 1) << (64 - bo));
    }
};

// RNE of a magnitude buf[0..n) (column of stride `stride`, LSB weight 2^e_lsb) to prec bits,
// stored in the ABI element format with sign `neg`.
// an output element's L limbs written as whole 16-byte vectors (one element's limbs are
// contiguous; limb-by-limb 8-byte stores from a warp left sectors half written in L2 and cost
// read-modify-write DRAM traffic)
MPC_DEV void store_limbs(uint64_t *dst, const uint64_t *v, int L) {
    if (!(L & 1) && !(reinterpret_cast<uintptr_t>(dst) & 15)) {
        for (int l = 0; l < L; l += 2) *reinterpret_cast<ulonglong2 *>(dst + l) = make_ulonglong2(v[l], v[l + 1]);
    } else {
        for (int l = 0; l < L; l++) dst[l] = v[l];
    }
}

MPC_DEV void round_store(const uint64_t *buf, int64_t stride, int n, int64_t e_lsb, bool neg, int prec, int L,
                         uint8_t *sign_out, int64_t *exp_out, uint64_t *limbs_out)
{
    // output limbs go out in pairs as they are formed (16-byte stores when aligned; no local array)
    const bool vec = !(L & 1) && !(reinterpret_cast<uintptr_t>(limbs_out) & 15);
    auto put2 = [&](int l, uint64_t a, uint64_t b) {
        if (vec) *reinterpret_cast<ulonglong2 *>(limbs_out + l) = make_ulonglong2(a, b);
        else { limbs_out[l] = a; if (l + 1 < L) limbs_out[l + 1] = b; }
    };
    int b = 0;
    for (int l = n - 1; l >= 0; l--) {
        const uint64_t v = buf[(int64_t)l * stride];
        if (v) { b = 64 * l + 64 - __clzll((long long)v); break; }
    }
    if (b == 0) {
        *sign_out = 0; *exp_out = 0;
        for (int l = 0; l < L; l += 2) put2(l, 0ull, 0ull);
        return;
    }
    const FixView F{buf, stride, n};
    int64_t E = e_lsb + b;
    const int64_t base = (int64_t)b - 64 * L;         // window = bits [b - 64L, b)
    const int drop = 64 * L - prec;
    // round bit = bit (b - prec - 1); sticky = OR of the bits below it
    const int64_t rpos = (int64_t)b - prec - 1;
    int rbit = 0, sticky = 0;
    if (rpos >= 0) {
        rbit = (int)((F.at(rpos >> 6) >> (rpos & 63)) & 1);
        const int64_t full = rpos >> 6;
        for (int64_t l = 0; l < full && !sticky; l++) if (F.at(l)) sticky = 1;
        if (!sticky && (rpos & 63) && (F.at(full) & ((1ull << (rpos & 63)) - 1))) sticky = 1;
    }
    const uint64_t w0 = F.bits64(base) & (drop ? ~((1ull << drop) - 1) : ~0ull);
    const int lsb = (int)((w0 >> drop) & 1);
    bool up = rbit && (sticky || lsb);
    if (up) {                                         // carry-out iff all kept bits are 1
        bool allones = (w0 | ((1ull << drop) - 1)) == ~0ull;
        for (int l = 1; l < L && allones; l++) allones = F.bits64(base + 64 * l) == ~0ull;
        if (allones) {
            for (int l = 0; l < L; l += 2) put2(l, 0ull, l + 1 == L - 1 ? (1ull << 63) : 0ull);
            if (L & 1) limbs_out[L - 1] = 1ull << 63;
            *sign_out = neg ? 1 : 0;
            *exp_out = E + 1;
            return;
        }
    }
    uint64_t c = up ? (1ull << drop) : 0ull;
    for (int l = 0; l < L; l += 2) {
        const uint64_t wa = l == 0 ? w0 : F.bits64(base + 64 * l);
        const uint64_t xa = wa + c;
        c = (xa < wa) ? 1ull : 0ull;
        uint64_t xb = 0;
        if (l + 1 < L) {
            const uint64_t wb = F.bits64(base + 64 * (l + 1));
            xb = wb + c;
            c = (xb < wb) ? 1ull : 0ull;
        }
        put2(l, xa, xb);
    }
    *sign_out = neg ? 1 : 0;
    *exp_out = E;
}

// two's complement fix[0..Lc) -> magnitude in place; returns the sign
MPC_DEV bool to_magnitude(uint64_t *fix, int64_t stride, int Lc) {
    const bool neg = (int64_t)fix[(int64_t)(Lc - 1) * stride] < 0;
    if (neg) {
        uint64_t c = 1;
        for (int l = 0; l < Lc; l++) {
            const uint64_t x = ~fix[(int64_t)l * stride] + c;
            c = (c && x == 0);
            fix[(int64_t)l * stride] = x;
        }
    }
    return neg;
}

// fix (two's complement, LSB weight 2^e0) -> RNE((-1)^alpha_neg fix 2^e0) in the ABI format
MPC_DEV void normalize_store(uint64_t *fix, int64_t stride, int Lc, int64_t e0, bool alpha_neg, int prec, int L,
                             uint8_t *sign_out, int64_t *exp_out, uint64_t *limbs_out)
{
    const bool neg = to_magnitude(fix, stride, Lc);
    round_store(fix, stride, Lc, e0, neg != alpha_neg, prec, L, sign_out, exp_out, limbs_out);
}


// NEXT-2: RNE(C0 + (-1)^alpha_neg V 2^e0), one rounding of the exact sum.  V = fix[0..Lc)
// (two's complement); the sum is formed in sign-magnitude in R = fix[Lc..Lc+Lw) over a window
// of 64 Lw >= 64 (Lc + L + 3) bits below the larger operand's top; bits of the smaller operand
// below the window collapse into a sticky LSB (>= 2 guard bits below the rounding position).
// C0 (N, L limbs, LSB weight 2^(exp - 64 L)) may alias the output element (read first).
MPC_DEV void accumulate_store(uint64_t *fix, int unused, int Lc, int Lw, int64_t e0, bool alpha_neg,
                              uint8_t c0s, int64_t c0e, const uint64_t *c0l, int prec, int L,
                              uint8_t *sign_out, int64_t *exp_out, uint64_t *limbs_out, int64_t stride, uint64_t *R)
{
    (void)unused;
    const bool sV = to_magnitude(fix, stride, Lc) != alpha_neg;
    int bV = 0;
    for (int l = Lc - 1; l >= 0; l--) {
        const uint64_t v = fix[(int64_t)l * stride];
        if (v) { bV = 64 * l + 64 - __clzll((long long)v); break; }
    }
    const bool cz = __ldg(c0l + L - 1) == 0;
    if (cz) { round_store(fix, stride, Lc, e0, sV, prec, L, sign_out, exp_out, limbs_out); return; }
    const bool sC = c0s != 0;
    const int64_t E1 = c0e - 64 * (int64_t)L;
    if (bV == 0) {                                    // C0 is already a prec-bit value
        uint64_t tmp[64];
        for (int l = 0; l < L; l++) tmp[l] = __ldg(c0l + l);
        *sign_out = sC ? 1 : 0; *exp_out = c0e;
        for (int l = 0; l < L; l++) limbs_out[l] = tmp[l];
        return;
    }
    const int64_t topV = e0 + bV, topC = c0e;
    const int64_t top = topV > topC ? topV : topC;
    int64_t WB = e0 < E1 ? e0 : E1;
    if (WB < top - 64 * (int64_t)Lw + 2) WB = top - 64 * (int64_t)Lw + 2;
    const FixView V{fix, stride, Lc};
    uint64_t cN[64];
    for (int l = 0; l < L; l++) cN[l] = __ldg(c0l + l);
    auto nbits = [&](int64_t pos) -> uint64_t {      // 64 bits of N from bit pos
        if (pos <= -64) return 0;
        if (pos < 0) return cN[0] << (-pos);
        const int64_t li = pos >> 6;
        const int bo = (int)(pos & 63);
        const uint64_t lo = li < L ? cN[li] : 0ull;
        if (!bo) return lo;
        const uint64_t hi = li + 1 < L ? cN[li + 1] : 0ull;
        return (lo >> bo) | (hi << (64 - bo));
    };
    auto below = [&](auto get, int nl, int64_t cut) -> bool {   // any bit below position cut
        if (cut <= 0) return false;
        const int64_t full = cut >> 6;
        for (int64_t l = 0; l < full && l < nl; l++) if (get(l)) return true;
        if (full < nl && (cut & 63) && (get(full) & ((1ull << (cut & 63)) - 1))) return true;
        return false;
    };
    const bool stV = below([&](int64_t l) { return V.at(l); }, Lc, WB - e0);
    const bool stC = below([&](int64_t l) { return l < L ? cN[l] : 0ull; }, L, WB - E1);
    // compare |X| and |Y| (aligned) from the top when subtracting
    const bool sub = sV != sC;
    bool xbig = true;
    if (sub) {
        int cmp = 0;
        for (int l = Lw - 1; l >= 0 && !cmp; l--) {
            uint64_t x = V.bits64(WB - e0 + 64 * (int64_t)l), y = nbits(WB - E1 + 64 * (int64_t)l);
            if (l == 0) { x |= stV; y |= stC; }
            cmp = x > y ? 1 : (x < y ? -1 : 0);
        }
        if (cmp == 0) { *sign_out = 0; *exp_out = 0; for (int l = 0; l < L; l++) limbs_out[l] = 0; return; }
        xbig = cmp > 0;
    }
    uint64_t c = 0;
    for (int l = 0; l < Lw; l++) {
        uint64_t x = V.bits64(WB - e0 + 64 * (int64_t)l), y = nbits(WB - E1 + 64 * (int64_t)l);
        if (l == 0) { x |= stV; y |= stC; }
        uint64_t r;
        if (!sub) { r = x + y + c; c = (r < x || (c && r == x)) ? 1 : 0; }
        else {
            const uint64_t a = xbig ? x : y, bb = xbig ? y : x;
            r = a - bb - c; c = (a < bb || (c && a == bb)) ? 1 : 0;
        }
        R[(int64_t)l * stride] = r;
    }
    const bool sR = sub ? (xbig ? sV : sC) : sV;
    round_store(R, stride, Lw, WB, sR, prec, L, sign_out, exp_out, limbs_out);
}

// The partial planes are streamed by a producer warp with cp.async.bulk: for each slot (in
// the fold's consumption order r = s+1..2, job, chunk) the strip partials[slot][i][j0 .. j0+COLS)
// lands in a shared-memory ring (PER slots per entry, RING entries), so ~RING*PER*COLS*4 bytes
// per block are in flight regardless of the consumers' registers.  COLS/2 consumer threads (two
// adjacent outputs each) walk a flat per-slot schedule (job of the slot, last slot of r) and run
// the carry chains; the fixed-point numbers live in shared memory, fix[part][limb][column].
constexpr int kFoldRing = 4;           // entries
constexpr int kFoldPer = 8;            // slots per entry
constexpr int kFoldEPT = 2;            // outputs per consumer thread (4: fewer instructions but slower, profiles/README.md)
static_assert(kFoldLdAlign % 4 == 0, "scratch pitch alignment");

template <int V> struct IntVec;
template <> struct IntVec<1> {
    MPC_DEV static void get_shared(uint32_t a, int32_t (&o)[1]) {
        asm volatile("ld.shared.s32 %0, [%1];" : "=r"(o[0]) : "r"(a) : "memory");
    }
};
template <> struct IntVec<2> {
    using T = int2;
    MPC_DEV static void get(const T &v, int32_t (&o)[2]) { o[0] = v.x; o[1] = v.y; }
    MPC_DEV static void get_shared(uint32_t a, int32_t (&o)[2]) {
        asm volatile("ld.shared.v2.s32 {%0, %1}, [%2];" : "=r"(o[0]), "=r"(o[1]) : "r"(a) : "memory");
    }
};
template <> struct IntVec<4> {
    using T = int4;
    MPC_DEV static void get(const T &v, int32_t (&o)[4]) { o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w; }
    MPC_DEV static void get_shared(uint32_t a, int32_t (&o)[4]) {
        asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(o[0]), "=r"(o[1]), "=r"(o[2]), "=r"(o[3]) : "r"(a) : "memory");
    }
};

// SFIX: the fixed-point limbs of the CTA's COLS outputs stay in shared memory, fix[part][limb][col]
// (no global round trip); otherwise (NEXT-2 sums, or s too large for shared memory) they go to
// the global scratch fix[part][limb][m*ldF]
// the EPT adjacent elements' words of one limb (16-byte stores for pairs)
// (GLOBAL: dst is the global scratch, stored with an L2 policy; else shared memory)
template <int EPT, bool GLOBAL>
MPC_DEV void store_ept(uint64_t *dst, const uint64_t *v, uint64_t pol) {
    if constexpr (!GLOBAL) {
        if constexpr (EPT == 1) { *dst = v[0]; }
        else {
#pragma unroll
            for (int x = 0; x < EPT; x += 2) *reinterpret_cast<ulonglong2 *>(dst + x) = make_ulonglong2(v[x], v[x + 1]);
        }
    } else if constexpr (EPT == 1) { st_global_u64_hint(dst, v[0], pol); }
    else {
#pragma unroll
        for (int x = 0; x < EPT; x += 2) st_global_v2u64_hint(dst + x, v[x], v[x + 1], pol);
    }
}

// TMAP: the producer fetches each ring entry (8 slots of one row's strip) with ONE 3-D TMA load
// (encode_partials_map) instead of 8 bulk copies -- the producer's instructions were a third of
// the kernel's; a short last entry over-reads into the next slots (never consumed)
// UNI1 (with TMAP): every (job, diagonal) has exactly one chunk (3 slots per diagonal, in job
// order), so a ring entry is one PAIR of diagonals (6 slots, one TMA load) and the consumers read
// it at fixed offsets: one wait and one release per pair, no per-slot bookkeeping
// UNIC (UPER > 0): the three jobs have equal chunk counts on every diagonal, so a diagonal's
// slots are groups of three (chunk c of job 0, 1, 2); a ring entry holds UPER / 3 whole groups and
// the consumers read a group at fixed offsets with one ring check per group instead of per slot
// MINB: CTAs per SM the register budget is sized for (7 for a grid just over one wave of 6:
// config 2's fold 56 -> 44 us; otherwise 6, as 7 spills a little)
template <int COLS, bool BETA, bool SFIX, int EPT = kFoldEPT, int RING = kFoldRing, bool TMAP = false, bool UNI1 = false,
          int UPER = 0, int MINB = 6>
__global__ void __launch_bounds__(COLS / EPT + 32, BETA ? 1 : (SFIX ? 3 : MINB))
fold_normalize_kernel(const FoldParams F, const __grid_constant__ CUtensorMap pmap)
{
    pdl_wait();
    constexpr bool UNIC = UPER > 0;
    static_assert(UPER % 3 == 0, "UNIC entries are whole groups of three slots");
    constexpr int PER = UNI1 ? 6 : UNIC ? UPER : kFoldPer;   // slots per ring entry
    constexpr int NCONS = COLS / EPT;                 // consumer threads
    extern __shared__ __align__(128) uint8_t fsm_raw[];
    if (F.drs && F.drs->status) return;              // device rule: s outside the planned range
    const int s = F.drs ? F.drs->cur.s : F.s;        // (device rule: the chosen plan's s, slots)
    const int32_t *const slotinfo = F.drs ? F.drs->cur.slotinfo : F.slotinfo;
    const int Lc0 = s / 8 + 3;                        // fixed-point limbs
    const int Lw = BETA ? Lc0 + F.L + 3 : 0;          // NEXT-2 sum window
    const int nslots = F.drs ? F.drs->cur.nslots : (int)F.nslots;
    int32_t *ring = reinterpret_cast<int32_t *>(fsm_raw);                                   // [RING][PER][COLS]
    uint16_t *cntq = reinterpret_cast<uint16_t *>(fsm_raw + RING * PER * COLS * 4);  // [job][s+2] chunk counts
    uint64_t *full = reinterpret_cast<uint64_t *>((reinterpret_cast<uintptr_t>(cntq + kMaxJobs * (s + 2)) + 15) & ~uintptr_t(15));
    uint64_t *empty = full + RING;
    uint64_t *fixs = empty + RING;               // SFIX: [2][Lc0][COLS] (16-byte aligned)
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    // chunk count of every (job, diagonal): the slots come in the order r = s+1..2, job, chunk
    for (int x = tid; x < kMaxJobs * (s + 2); x += blockDim.x)
        cntq[x] = (uint16_t)((x % (s + 2)) < 2 ? 0 : slotinfo[x * 2 + 1]);
    if (tid == 0) {
        for (int e = 0; e < RING; e++) { mbar_init(&full[e], 1); mbar_init(&empty[e], NCONS / 32); }
        fence_barrier_init();
    }
    __syncthreads();
    // block (x, y): row i = (y / nsub) * 128 + x, columns j0 = (y % nsub) * COLS, so the 128
    // blocks of one (row block, strip) are adjacent in launch order
    // (a 1-D grid: block b = y * 128 + x)
    const int64_t nsub = (F.n + COLS - 1) / COLS;
    const int64_t bx = (int64_t)blockIdx.x & (kRowBlk - 1), by = (int64_t)blockIdx.x >> 7;
    const int64_t i = (by / nsub) * kRowBlk + bx;
    const int64_t j0 = (by % nsub) * COLS;            // COLS divides the 256-column strip
    if (i >= F.m) return;
    // NEXT-4: this row's triangle d = sr <= s; its diagonals r = sr+1 .. 2 are the slots from
    // the first slot of (job 0, r = sr+1) on (slots of larger r are not read)
    const int sr = F.sblk ? F.sblk[i >> kSBlkShift] : s;
    const int sl0 = sr == s ? 0 : slotinfo[(sr + 1) * 2];
    if (warp == NCONS / 32) {
        // ---------------- producer warp
        if (lane == 0 && TMAP) {
            static_assert(!TMAP || COLS == kStrip, "TMA entries are whole strips");
            const int g0 = (int)((((i >> 7) * F.nstrips + (j0 >> 8)) * nslots));   // global slot of slot 0
            const int row = (int)(i & (kRowBlk - 1));
            int e = 0; uint32_t ph = 0;
            // partial planes are read once: evict-first, so the fixed-point scratch stays in L2
            const uint64_t ppol = F.l2hint ? l2_policy_evict_first() : l2_policy_evict_normal();
            for (int sl = sl0; sl < nslots; sl += PER) {
                mbar_wait(&empty[e], ph ^ 1);
                mbar_arrive_expect_tx(&full[e], (uint32_t)(PER * COLS * 4));
                tma_load_3d_hint(ring + e * PER * COLS, &pmap, &full[e], 0, row, g0 + sl, ppol);
                if (++e == RING) { e = 0; ph ^= 1; }
            }
        } else if (lane == 0) {
            const int32_t *region = F.partials + part_off(i, j0, 0, nslots, F.nstrips);   // slot 0
            int e = 0; uint32_t ph = 0;
            for (int sl = sl0; sl < nslots; sl += PER) {
                const int cnt = nslots - sl < PER ? nslots - sl : PER;
                mbar_wait(&empty[e], ph ^ 1);
                mbar_arrive_expect_tx(&full[e], (uint32_t)(cnt * COLS * 4));
                for (int f = 0; f < cnt; f++)                // slot blocks are kTileElems apart
                    bulk_load(ring + (e * PER + f) * COLS, region + (int64_t)(sl + f) * kTileElems, COLS * 4, &full[e]);
                if (++e == RING) { e = 0; ph ^= 1; }
            }
        }
        return;
    }
    // ---------------- consumers: outputs j0 + EPT tid .. + EPT-1.  The fixed-point limbs go to
    // the global scratch fix[part][limb][m*ldF] (column = element), read back by the rounding.
    const int col = EPT * tid;
    const int64_t jj = j0 + col;                      // first of the EPT elements
    // the fixed-point scratch is read back by the same thread at the end: keep it in L2
    const uint64_t fpol = F.l2hint ? l2_policy_evict_last() : l2_policy_evict_normal();
    const int64_t lstride = SFIX ? (int64_t)COLS : F.m * F.ldF;   // limb stride
    uint64_t *fixg = SFIX ? fixs + col : F.fix + i * F.ldF + jj;
    int64_t t0[EPT], t1[EPT], t2[EPT];
    int64_t cr[2][EPT];                               // [part][element] carries
    uint64_t cur[2][EPT];
#pragma unroll
    for (int x = 0; x < EPT; x++) { t0[x] = t1[x] = t2[x] = 0; cr[0][x] = cr[1][x] = 0; cur[0][x] = cur[1][x] = 0; }
    int e = 0, fill = 0; uint32_t ph = 0;
    const bool live = jj < F.n;                       // (the rest of the EPT too: ldF is a multiple of EPT)
    // next slot's strip from the ring (consumer side of the producer's bulk copies)
    // the ring's slots are consecutive COLS-int32 rows: this thread's column advances by one row
    // per slot (a shared-space address, no per-slot index arithmetic) and wraps with the ring
    const uint32_t ring0 = smem_u32(ring) + (uint32_t)col * 4u;
    uint32_t addr = ring0;
    // Releasing a ring entry: the producer's next write into it is an ASYNC-proxy write (TMA / bulk
    // copy), which the mbarrier hand-off alone does not order after this warp's generic-proxy shared
    // loads (the last of which may still be in flight): each lane fences the proxies first.  Without
    // the fence ~5-10 % of config-4 folds corrupted a few outputs (tools/determinism.py, MPCGEMM_DBG=16).
    auto release = [&]() {
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[e]);
    };
    auto next = [&](int32_t (&v)[EPT]) {
        if (fill == 0) mbar_wait(&full[e], ph);
        IntVec<EPT>::get_shared(addr, v);
        addr += (uint32_t)COLS * 4u;
        if (++fill == PER) {
            fill = 0;
            release();
            if (++e == RING) { e = 0; ph ^= 1; addr = ring0; }
        }
    };
    // diagonals r = sr+1 .. 2 (byte b = sr + 1 - r of the fixed-point number), two per iteration:
    //   acc = carry + D_b + 256 D_{b+1};  emit 16 bits at bit 8 b;  carry = acc >> 16
    // D_r: the chunk sums of the jobs' partials combined by Eq. 6 (3M) or Eq. 5 (4M)
    auto diag = [&](int r, int64_t (&d)[2][EPT]) {
        int64_t u0[EPT], u1[EPT], u2[EPT];
#pragma unroll
        for (int x = 0; x < EPT; x++) u0[x] = u1[x] = u2[x] = 0;
        int32_t v[EPT];
        if constexpr (UNI1) {                         // the entry is resident: three fixed slots
            int32_t w1[EPT], w2[EPT];
            IntVec<EPT>::get_shared(addr, v);
            IntVec<EPT>::get_shared(addr + (uint32_t)COLS * 4u, w1);
            IntVec<EPT>::get_shared(addr + (uint32_t)COLS * 8u, w2);
            addr += (uint32_t)COLS * 12u;
#pragma unroll
            for (int x = 0; x < EPT; x++) { u0[x] = v[x]; u1[x] = w1[x]; u2[x] = w2[x]; }
        } else if constexpr (UNIC) {                  // c groups (chunk c of jobs 0, 1, 2)
            for (int c = cntq[r]; c > 0; c--) {
                int32_t w1[EPT], w2[EPT];
                if (fill == 0) mbar_wait(&full[e], ph);
                IntVec<EPT>::get_shared(addr, v);
                IntVec<EPT>::get_shared(addr + (uint32_t)COLS * 4u, w1);
                IntVec<EPT>::get_shared(addr + (uint32_t)COLS * 8u, w2);
                addr += (uint32_t)COLS * 12u;
#pragma unroll
                for (int x = 0; x < EPT; x++) { u0[x] += v[x]; u1[x] += w1[x]; u2[x] += w2[x]; }
                fill += 3;
                if (fill == PER) {
                    fill = 0;
                    release();
                    if (++e == RING) { e = 0; ph ^= 1; addr = ring0; }
                }
            }
        } else {                                      // slots in the order (job, chunk)
            for (int c = cntq[r]; c > 0; c--) {
                next(v);
#pragma unroll
                for (int x = 0; x < EPT; x++) u0[x] += v[x];
            }
            for (int c = cntq[(s + 2) + r]; c > 0; c--) {
                next(v);
#pragma unroll
                for (int x = 0; x < EPT; x++) u1[x] += v[x];
            }
            for (int c = cntq[2 * (s + 2) + r]; c > 0; c--) {
                next(v);
#pragma unroll
                for (int x = 0; x < EPT; x++) u2[x] += v[x];
            }
        }
#pragma unroll
        for (int x = 0; x < EPT; x++) {
            if (F.method == 3) { d[0][x] = u0[x] - u1[x]; d[1][x] = u2[x] - u0[x] - u1[x]; }   // Eq. 6
            else               { d[0][x] = u0[x] - u1[x]; d[1][x] = u2[x]; }                   // Eq. 5
        }
    };
    // limb pointers advance by one limb stride per completed 64-bit limb (no index arithmetic)
    uint64_t *lp0 = fixg, *lp1 = fixg + (int64_t)Lc0 * lstride;
    int b = 0, r = sr + 1;
    // UNI1: wait for / release one ring entry (a pair of diagonals)
    auto entry_begin = [&]() {
        if constexpr (UNI1) { mbar_wait(&full[e], ph); addr = ring0 + (uint32_t)(e * PER * COLS * 4); }
    };
    auto entry_end = [&]() {
        if constexpr (UNI1) {
            release();
            if (++e == RING) { e = 0; ph ^= 1; }
        }
    };
    for (; r >= 3; r -= 2, b += 2) {
        int64_t d[2][EPT];
        entry_begin();
        diag(r, d);
#pragma unroll
        for (int p = 0; p < 2; p++)
#pragma unroll
            for (int x = 0; x < EPT; x++) cr[p][x] += d[p][x];                  // carry + D_b
        diag(r - 1, d);
        entry_end();
        const int sh = 8 * (b & 7);
#pragma unroll
        for (int p = 0; p < 2; p++)
#pragma unroll
            for (int x = 0; x < EPT; x++) {
                const int64_t acc = cr[p][x] + d[p][x] * 256;
                cur[p][x] |= (uint64_t)(acc & 0xFFFF) << sh;
                cr[p][x] = acc >> 16;
            }
        if ((b & 7) == 6) {                           // a 64-bit limb complete
            if (live) { store_ept<EPT, !SFIX>(lp0, cur[0], fpol); store_ept<EPT, !SFIX>(lp1, cur[1], fpol); }
            lp0 += lstride; lp1 += lstride;
#pragma unroll
            for (int x = 0; x < EPT; x++) cur[0][x] = cur[1][x] = 0;
        }
    }
    if (r == 2) {                                     // odd number of diagonals: the last one alone
        int64_t d0[2][EPT];
        entry_begin();
        diag(2, d0);
        entry_end();
        const int sh = 8 * (b & 7);
#pragma unroll
        for (int p = 0; p < 2; p++)
#pragma unroll
            for (int x = 0; x < EPT; x++) {
                const int64_t acc = cr[p][x] + d0[p][x];
                cur[p][x] |= (uint64_t)(acc & 0xFF) << sh;
                cr[p][x] = acc >> 8;
            }
        b++;
    }
    // the rounding reads each (element, part)'s limbs from a shared-memory column carved out of the
    // ring, which is free once every consumer is past its last diagonal (dynamic limb indexing on
    // a thread-local copy went to local memory, ~a third of the fold's stall samples at config 4)
    constexpr int RING_BYTES = RING * PER * COLS * 4;
    const bool smem_norm = !BETA && !SFIX && Lc0 * NCONS * 8 <= RING_BYTES && !F.norm_generic;
    if (smem_norm) asm volatile("bar.sync 1, %0;" ::"r"(NCONS) : "memory");
    if (!live) return;
    // the final carries at bit 8 sr, sign-extended to Lc0 limbs
    const int l0 = sr >> 3, o = 8 * (sr & 7);
#pragma unroll
    for (int p = 0; p < 2; p++) {
        uint64_t w[EPT][2];
#pragma unroll
        for (int x = 0; x < EPT; x++) {
            const uint64_t c = (uint64_t)cr[p][x], sx = cr[p][x] < 0 ? ~0ull : 0ull;
            w[x][0] = cur[p][x] | (c << o);
            w[x][1] = o ? ((c >> (64 - o)) | (sx << o)) : sx;
        }
        uint64_t *fx = fixg + (int64_t)p * Lc0 * lstride;
        uint64_t w0[EPT], w1[EPT], sx[EPT];
#pragma unroll
        for (int x = 0; x < EPT; x++) { w0[x] = w[x][0]; w1[x] = w[x][1]; sx[x] = cr[p][x] < 0 ? ~0ull : 0ull; }
        store_ept<EPT, !SFIX>(fx + (int64_t)l0 * lstride, w0, fpol);
        store_ept<EPT, !SFIX>(fx + (int64_t)(l0 + 1) * lstride, w1, fpol);
        for (int l = l0 + 2; l < Lc0; l++) store_ept<EPT, !SFIX>(fx + (int64_t)l * lstride, sx, fpol);
    }
#pragma unroll 1
    for (int x = 0; x < EPT; x++) {
        const int64_t j = jj + x;
        if (j >= F.n) break;
        uint64_t *f0 = fixg + x, *f1 = fixg + x + (int64_t)(Lc0 + Lw) * lstride;   // parts: [0, Lc0+Lw), [Lc0+Lw, ..)
        if (BETA) f1 = fixg + x + (int64_t)Lc0 * lstride;
        const int64_t e0 = F.eA[i] + F.eB[j] + 6 - 8 * (int64_t)(sr + 1);
        const int64_t oi = i * F.Cre.ld + j;
        const int64_t oj = i * F.Cim.ld + j;
        if (BETA) {
            uint64_t *R0 = F.fix + 2 * (int64_t)Lc0 * lstride + i * F.ldF + j;          // sum windows
            const int64_t ci = i * F.C0re.ld + j, cj = i * F.C0im.ld + j;
            const uint8_t s0 = F.C0re.sign[ci], s1 = F.C0im.sign[cj];   // read before the (aliasing) write
            const int64_t x0 = F.C0re.exp[ci], x1 = F.C0im.exp[cj];
            accumulate_store(f0, (int)0, Lc0, Lw, e0, F.alpha_neg, s0, x0, F.C0re.limbs + ci * F.L, F.prec, F.L,
                             F.Cre.sign + oi, F.Cre.exp + oi, F.Cre.limbs + oi * F.L, lstride, R0);
            accumulate_store(f1, (int)0, Lc0, Lw, e0, F.alpha_neg, s1, x1, F.C0im.limbs + cj * F.L, F.prec, F.L,
                             F.Cim.sign + oj, F.Cim.exp + oj, F.Cim.limbs + oj * F.L, lstride, R0);
        } else if (SFIX) {                            // limbs in shared memory: round in place
#pragma unroll 1
            for (int p = 0; p < 2; p++) {
                const DMatOut &Co = p ? F.Cim : F.Cre;
                const int64_t oo = p ? oj : oi;
                normalize_store(fixg + x + (int64_t)p * Lc0 * lstride, lstride, Lc0, e0, F.alpha_neg, F.prec, F.L,
                                Co.sign + oo, Co.exp + oo, Co.limbs + oo * F.L);
            }
        } else {
            // copy each part's limbs to a thread-local array with independent (batched) loads,
            // then magnitude + RNE on the L1-resident copy (the scratch reads were a dependent
            // chain of global loads -- profiles/ncu_hbm_r1o.md)
            if (smem_norm) {
                uint64_t *colp = reinterpret_cast<uint64_t *>(ring) + tid;   // [limb][consumer]
#pragma unroll 1
                for (int p = 0; p < 2; p++) {
                    const uint64_t *src = fixg + x + (int64_t)p * Lc0 * lstride;
#pragma unroll 8
                    for (int l = 0; l < Lc0; l++) colp[l * NCONS] = src[(int64_t)l * lstride];
                    const DMatOut &Co = p ? F.Cim : F.Cre;
                    const int64_t oo = p ? oj : oi;
                    normalize_store(colp, NCONS, Lc0, e0, F.alpha_neg, F.prec, F.L, Co.sign + oo, Co.exp + oo, Co.limbs + oo * F.L);
                }
                continue;
            }
            uint64_t loc[kMaxSlices / 8 + 3];
#pragma unroll 1
            for (int p = 0; p < 2; p++) {
                const uint64_t *src = fixg + x + (int64_t)p * Lc0 * lstride;
#pragma unroll 8
                for (int l = 0; l < Lc0; l++) loc[l] = src[(int64_t)l * lstride];
                const DMatOut &Co = p ? F.Cim : F.Cre;
                const int64_t oo = p ? oj : oi;
                normalize_store(loc, 1, Lc0, e0, F.alpha_neg, F.prec, F.L, Co.sign + oo, Co.exp + oo, Co.limbs + oo * F.L);
            }
        }
    }
}

size_t fold_smem(int s, int cols, bool sfix, int ring = kFoldRing, int per = kFoldPer) {
    const size_t base = (size_t)ring * per * cols * 4 + 2 * (size_t)kMaxJobs * (s + 2) + 32 + (size_t)2 * ring * 8 + 16;
    return base + (sfix ? (size_t)2 * (s / 8 + 3) * cols * 8 + 16 : 0);
}

// shared-memory-limbs fold: 128 columns per CTA, one output per consumer thread, an 8-entry ring
// (3 CTAs per SM: ~96 KB of partial strips in flight per SM) -- or, when the limbs do not fit,
// the global scratch
constexpr int kSfixCols = 128, kSfixRing = 8;
static bool fold_sfix(int s, bool beta) {
    // measured slower (fewer resident consumer threads: the fold is issue-bound), so off by default
    if (beta || !getenv("MPCGEMM_FOLD_SFIX")) return false;
    return fold_smem(s, kSfixCols, true, kSfixRing) <= 220 * 1024;
}

template <int COLS, bool BETA, bool SFIX, int EPT, int RING, bool TMAP = false, bool UNI1 = false, int UPER = 0, int MINB = 6>
static cudaError_t fold_launch_t(const FoldParams &F, cudaStream_t st) {
    constexpr int PER = UNI1 ? 6 : UPER > 0 ? UPER : kFoldPer;
    const size_t sm = fold_smem(F.s, COLS, SFIX, RING, PER);
    auto kern = fold_normalize_kernel<COLS, BETA, SFIX, EPT, RING, TMAP, UNI1, UPER, MINB>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    const int64_t blocks = (int64_t)kRowBlk * ((F.n + COLS - 1) / COLS) * ((F.m + kRowBlk - 1) / kRowBlk);
    if (blocks > INT_MAX) return cudaErrorInvalidValue;
    alignas(64) uint8_t map[128] = {};
    if (TMAP) {
        // the partial planes of all (row block, strip) pairs: nslots is the launch's (the device
        // rule's plans have at most F.nslots slots and share the layout's base)
        const int64_t gslots = ((F.m + kRowBlk - 1) / kRowBlk) * F.nstrips * F.nslots;
        if (encode_partials_map(map, F.partials, gslots, PER)) return cudaErrorInvalidValue;
    }
    return launch_pdl(kern, dim3((unsigned)blocks), dim3(COLS / EPT + 32), sm, st, F,
                      *reinterpret_cast<const CUtensorMap *>(map));
}

cudaError_t fold_normalize_launch(const FoldParams &F, cudaStream_t st)
{
    if (F.m == 0 || F.n == 0) return cudaSuccess;
    if (F.s > kMaxSlices || (F.ldF % kFoldEPT)) return cudaErrorInvalidValue;
    // (device rule: F.nslots is the largest candidate's slot count, so the map covers the chosen plan)
    const bool tmap = !getenv("MPCGEMM_FOLD_BULK");
    const bool uni1 = tmap && F.uni1 && !getenv("MPCGEMM_FOLD_NOUNI1");
    // F.unic: the plan's slots are in (chunk, job) order -- only the UNIC consumer reads that
    // order (the plan chose it only if MPCGEMM_FOLD_UNIC != 0 and no MPCGEMM_FOLD_SFIX); the entry
    // size is 6 (default), 9 or 12 slots
    const char *ue = getenv("MPCGEMM_FOLD_UNIC");
    const int unic = F.unic && !uni1 ? (tmap && ue && (atoi(ue) == 9 || atoi(ue) == 12) ? atoi(ue) : 6) : 0;
    if (F.beta) return uni1 ? fold_launch_t<256, true, false, kFoldEPT, 5, true, true>(F, st)
                     : unic ? (tmap ? fold_launch_t<256, true, false, kFoldEPT, 5, true, false, 6>(F, st)
                                    : fold_launch_t<256, true, false, kFoldEPT, 5, false, false, 6>(F, st))
                     : tmap ? fold_launch_t<256, true, false, kFoldEPT, kFoldRing, true>(F, st)
                            : fold_launch_t<256, true, false, kFoldEPT, kFoldRing>(F, st);
    if (!unic && fold_sfix(F.s, false)) return fold_launch_t<kSfixCols, false, true, 1, kSfixRing>(F, st);
    if (uni1) {
        // a grid just over one wave of 6 CTAs per SM runs in one wave of 7
        static int nsm = 0;
        if (!nsm) { int dev = 0; cudaGetDevice(&dev); cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev); }
        const int64_t blocks = (int64_t)kRowBlk * ((F.n + 255) / 256) * ((F.m + kRowBlk - 1) / kRowBlk);
        if (blocks > 6LL * nsm && blocks <= 7LL * nsm && !getenv("MPCGEMM_FOLD_NO7"))
            return fold_launch_t<256, false, false, kFoldEPT, 5, true, true, 0, 7>(F, st);
    }
    return uni1 ? fold_launch_t<256, false, false, kFoldEPT, 5, true, true>(F, st)
         : unic == 12 ? fold_launch_t<256, false, false, kFoldEPT, 3, true, false, 12>(F, st)
         : unic == 9 ? fold_launch_t<256, false, false, kFoldEPT, 4, true, false, 9>(F, st)
         : unic ? (tmap ? fold_launch_t<256, false, false, kFoldEPT, 5, true, false, 6>(F, st)
                        : fold_launch_t<256, false, false, kFoldEPT, 5, false, false, 6>(F, st))
         : tmap ? fold_launch_t<256, false, false, kFoldEPT, kFoldRing, true>(F, st)
                : fold_launch_t<256, false, false, kFoldEPT, kFoldRing>(F, st);
}

// fixed-point scratch size (uint64 words) for the fold (0 when the limbs stay in shared memory)
size_t fold_scratch_words(int64_t m, int64_t ldF, int s, int L, bool beta) {
    if (fold_sfix(s, beta)) return 0;
    const int Lc0 = s / 8 + 3;
    return (size_t)m * ldF * (2 * Lc0 + (beta ? Lc0 + L + 3 : 0));
}

__global__ void zero_output_kernel(DMatOut C, int64_t m, int64_t n, int L) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    for (int64_t i = blockIdx.y; i < m; i += gridDim.y) {
        const int64_t o = i * C.ld + j;
        C.sign[o] = 0; C.exp[o] = 0;
        for (int l = 0; l < L; l++) C.limbs[o * L + l] = 0;
    }
}

cudaError_t zero_output_launch(DMatOut C, int64_t m, int64_t n, int L, cudaStream_t st) {
    if (m == 0 || n == 0) return cudaSuccess;
    dim3 grid((unsigned)((n + 127) / 128), (unsigned)(m < 65535 ? m : 65535));
    zero_output_kernel<<<grid, 128, 0, st>>>(C, m, n, L);
    return cudaGetLastError();
}

}  // namespace mpc
