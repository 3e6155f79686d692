// lu.cu -- NEXT-3: the kernels of the blocked right-looking complex LU with partial pivoting
// (Fig. 3) and of the Eq. 7 solve.  The trailing update A22 -= L21 U12 is
// the Ozaki GEMM of this library (mpcgemm.cu, accumulate mode); these kernels do the panel
// (xGETF2: pivot search, row swap, reciprocal, column scaling, rank-1 updates), U12 := L11^-1
// A12 and the substitutions, every scalar operation MPC-style (mpscalar.cuh).
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#include "common.cuh"
#include "kernels.h"
#include "mpscalar.cuh"
#include "mpwarp.cuh"

// resident blocks per SM for the thread-per-part rank-1 update (large launches): capping it at
// 128 registers doubles the threads in flight; measured best (3: 170, 6: 85 registers are slower)
#ifndef MPC_UPD_MINB
#define MPC_UPD_MINB 4
#endif
namespace mpc {

using namespace mps;

struct El {                 // pointers to one real element
    uint8_t *s; int64_t *e; uint64_t *l;
};
MPC_DEV El el(int L, const DMatOut &M, int64_t r, int64_t c) {
    const int64_t i = r * M.ld + c;
    return El{M.sign + i, M.exp + i, M.limbs + i * L};
}
template <int C>
MPC_DEV Num<C> ld(int L, const El &x) { return load<C>(L, x.s, x.e, x.l); }

// ---------------------------------------------------------------- pivot search (one CTA)
// the larger key, ties to the smaller row (the first maximum)
MPC_DEV void key_max(int64_t &e, double &v, int64_t &r, int64_t e2, double v2, int64_t r2) {
    const Key a{e, v}, b{e2, v2};
    if (key_greater(b, a) || (!key_greater(a, b) && r2 < r)) { e = e2; v = v2; r = r2; }
}

__global__ void __launch_bounds__(1024) lu_pivot_kernel(int L, DMatOut re, DMatOut im, int64_t n, int64_t c, int64_t *ipiv)
{
    __shared__ int64_t se[32], sr[32];
    __shared__ double sv[32];
    Key best; best.e = INT64_MIN; best.v = 0.0;
    int64_t br = c;
    for (int64_t r = c + threadIdx.x; r < n; r += blockDim.x) {
        const El a = el(L, re, r, c), b = el(L, im, r, c);
        const Key k = pivot_key(a.s, a.e, a.l, b.s, b.e, b.l, L);
        if (key_greater(k, best)) { best = k; br = r; }      // rows ascending: first max kept
    }
    int64_t e = best.e, r = br;
    double v = best.v;
    for (int o = 16; o > 0; o >>= 1)                        // warp, then across warps
        key_max(e, v, r, __shfl_xor_sync(0xFFFFFFFFu, e, o), __shfl_xor_sync(0xFFFFFFFFu, v, o),
                __shfl_xor_sync(0xFFFFFFFFu, r, o));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    if (lane == 0) { se[warp] = e; sv[warp] = v; sr[warp] = r; }
    __syncthreads();
    if (warp) return;
    e = lane < nw ? se[lane] : INT64_MIN; v = lane < nw ? sv[lane] : 0.0; r = lane < nw ? sr[lane] : n;
    for (int o = 16; o > 0; o >>= 1)
        key_max(e, v, r, __shfl_xor_sync(0xFFFFFFFFu, e, o), __shfl_xor_sync(0xFFFFFFFFu, v, o),
                __shfl_xor_sync(0xFFFFFFFFu, r, o));
    if (lane == 0) ipiv[c] = r;
}

// ---------------------------------------------------------------- row swap (all columns)
// one thread per (column, part, limb): every word of the two rows moves independently (a
// per-element loop over the limbs was a chain of dependent load/store pairs, ~8 us per column)
__global__ void lu_swap_kernel(int L, DMatOut re, DMatOut im, int64_t ncols, int64_t c, const int64_t *ipiv)
{
    const int64_t p = ipiv[c];
    if (p == c) return;
    const int64_t per = 2 * (int64_t)L;               // words per column (both parts)
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < ncols * per; g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = g / per;
        const int w = (int)(g - t * per);
        const int part = w >= L;
        const int l = w - part * L;
        const DMatOut &M = part ? im : re;
        uint64_t *a = M.limbs + (c * M.ld + t) * L + l, *b = M.limbs + (p * M.ld + t) * L + l;
        const uint64_t x = *a, y = *b;
        *a = y; *b = x;
        if (l == 0) {
            const int64_t ia = c * M.ld + t, ib = p * M.ld + t;
            const uint8_t sa = M.sign[ia], sb = M.sign[ib];
            const int64_t ea = M.exp[ia], eb = M.exp[ib];
            M.sign[ia] = sb; M.sign[ib] = sa; M.exp[ia] = eb; M.exp[ib] = ea;
        }
    }
}

// Every MP-arithmetic kernel below gives the two real parts of a complex result to the two
// lanes of a lane pair (part = lane & 1): each lane computes one exactly rounded part
// (cfms_part / crecip_part), halving the per-element latency chain.

// ---------------------------------------------------------------- reciprocal of the pivot
// scratch: sign[2], exp[2], limbs[2][L] (re, im of 1 / A_cc); *info = c + 1 on the first zero
template <int C>
__global__ void lu_recip_kernel(int L, DMatOut re, DMatOut im, int64_t c, int prec, uint8_t *rs, int64_t *rexp,
                                uint64_t *rl, int32_t *info)
{
    const int part = threadIdx.x;
    if (part > 1 || blockIdx.x) return;
    const Num<C> zr = ld<C>(L, el(L, re, c, c)), zi = ld<C>(L, el(L, im, c, c));
    if (zr.zero && zi.zero) {
        if (part == 0 && info && *info == 0) *info = (int32_t)(c + 1);
        rs[part] = 0; rexp[part] = 0;
        for (int q = 0; q < L; q++) rl[part * L + q] = 0;
        return;
    }
    crecip_part<C>(L, part, zr, zi, prec, rs + part, rexp + part, rl + part * L);
}

// store one computed part (after both lanes of the pair have read their inputs)
MPC_DEV void put_part(const El &o, uint8_t s_, int64_t e_, const uint64_t *l_, int L) {
    *o.s = s_; *o.e = e_;
    for (int q = 0; q < L; q++) o.l[q] = l_[q];
}

// ---------------------------------------------------------------- column scaling
// A_rc := cmul(A_rc, 1 / A_cc) for r in [r0, r1)   (in place: the pair syncs before storing)
template <int C>
__global__ void __launch_bounds__(128) lu_scale_kernel(int L, DMatOut re, DMatOut im, int64_t r0, int64_t r1, int64_t c,
                                                       int prec, const uint8_t *rs, const int64_t *rexp,
                                                       const uint64_t *rl)
{
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int part = (int)(g & 1);
    const int64_t r = r0 + (g >> 1);
    if (r >= r1) return;                               // both lanes of a pair leave together
    const Num<C> yr = load<C>(L, rs, rexp, rl), yi = load<C>(L, rs + 1, rexp + 1, rl + L);
    const El a = el(L, re, r, c), b = el(L, im, r, c);
    const Num<C> xr = ld<C>(L, a), xi = ld<C>(L, b);
    uint8_t so; int64_t eo; uint64_t lo[C];
    cfms_part<C>(L, part, nullptr, xr, xi, yr, yi, prec, &so, &eo, lo);
    __syncwarp(3u << (threadIdx.x & 30));
    put_part(part ? b : a, so, eo, lo, L);
}

// ---------------------------------------------------------------- warp-cooperative (L <= 12)
// one warp per (element, part), one limb per lane (mpwarp.cuh)
MPC_DEV mpw::WNum wld(int L, const DMatOut &M, int64_t r, int64_t c, int lane) {
    const El x = el(L, M, r, c);
    return mpw::wload(L, x.s, x.e, x.l, lane);
}

// A_rc := cmul(A_rc, 1 / A_cc), r in [r0, r1): 4 elements per 256-thread block; every warp has
// its operands in registers (block barrier) before any warp stores (in place)
__global__ void __launch_bounds__(256) lu_scale_wkernel(int L, DMatOut re, DMatOut im, int64_t r0, int64_t r1, int64_t c,
                                                        int prec, const uint8_t *rs, const int64_t *rexp,
                                                        const uint64_t *rl)
{
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, part = warp & 1;
    const int64_t r = r0 + (int64_t)blockIdx.x * 4 + (warp >> 1);
    const bool on = r < r1;
    mpw::WNum xr{}, xi{}, yr{}, yi{};
    if (on) {
        xr = wld(L, re, r, c, lane); xi = wld(L, im, r, c, lane);
        yr = mpw::wload(L, rs, rexp, rl, lane); yi = mpw::wload(L, rs + 1, rexp + 1, rl + L, lane);
    }
    __syncthreads();
    if (!on) return;
    const El o = el(L, part ? im : re, r, c);
    mpw::cfms_warp(L, part, false, xr, xr, xi, yr, yi, prec, o.s, o.e, o.l, lane);
}

// A_rt := cfms(A_rt, A_rc, A_ct), r in [r0, r1), t in [t0, t1): one warp per (r, t, part)
__global__ void __launch_bounds__(256) lu_update_wkernel(int L, DMatOut re, DMatOut im, int64_t r0, int64_t r1, int64_t t0,
                                                         int64_t t1, int64_t c, int prec)
{
    const int lane = threadIdx.x & 31;
    const int64_t nt = t1 - t0, total = (r1 - r0) * nt * 2;
    for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < total;
         w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int part = (int)(w & 1);
        const int64_t e = w >> 1, r = r0 + e / nt, t = t0 + e % nt;
        const mpw::WNum lr = wld(L, re, r, c, lane), li = wld(L, im, r, c, lane);
        const mpw::WNum ur = wld(L, re, c, t, lane), ui = wld(L, im, c, t, lane);
        const El a = el(L, part ? im : re, r, t);
        const mpw::WNum av = mpw::wload(L, a.s, a.e, a.l, lane);
        __syncwarp();
        mpw::cfms_warp(L, part, true, av, lr, li, ur, ui, prec, a.s, a.e, a.l, lane);
    }
}

// ---------------------------------------------------------------- rank-1 update
// A_rt := cfms(A_rt, A_rc, A_ct) for r in [r0, r1), t in [t0, t1)  (lane pairs: the two parts)
template <int C>
__global__ void __launch_bounds__(128, MPC_UPD_MINB) lu_update_kernel(int L, DMatOut re, DMatOut im, int64_t r0, int64_t r1, int64_t t0,
                                                        int64_t t1, int64_t c, int prec)
{
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int part = (int)(g & 1);
    const int64_t t = t0 + (g >> 1);
    if (t >= t1) return;
    const Num<C> ur = ld<C>(L, el(L, re, c, t)), ui = ld<C>(L, el(L, im, c, t));
    const DMatOut &T = part ? im : re;
    for (int64_t r = r0 + blockIdx.y; r < r1; r += gridDim.y) {
        const Num<C> lr = ld<C>(L, el(L, re, r, c)), li = ld<C>(L, el(L, im, r, c));
        const El a = el(L, T, r, t);
        const Num<C> av = ld<C>(L, a);
        cfms_part<C>(L, part, &av, lr, li, ur, ui, prec, a.s, a.e, a.l);
    }
}

// ---------------------------------------------------------------- Eq. 7 solve
// B (n x nrhs) := U^-1 L^-1 P B with the factors above, one launch per substitution step:
//   all reciprocals 1 / U_cc at once (they do not depend on B); the row swaps in order;
//   forward  c = 0..n-2:  B_rq := cfms(B_rq, L_rc, B_cq)                     (r > c)
//   backward c = n-1..0:  x = cmul(B_cq, 1/U_cc); X_cq := x; B_rq := cfms(B_rq, U_rc, x) (r < c)
//   (every thread of step c recomputes x from the unchanged B_cq; X holds the solution rows,
//   copied back to B at the end)
template <int C>
__global__ void lu_recip_all_kernel(int L, DMatOut fre, DMatOut fim, int64_t n, int prec, DMatOut rre, DMatOut rim)
{
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int part = (int)(g & 1);
    const int64_t c = g >> 1;
    if (c >= n) return;
    const Num<C> zr = ld<C>(L, el(L, fre, c, c)), zi = ld<C>(L, el(L, fim, c, c));
    const El o = el(L, part ? rim : rre, 0, c);
    if (zr.zero && zi.zero) {
        *o.s = 0; *o.e = 0;
        for (int q = 0; q < L; q++) o.l[q] = 0;
        return;
    }
    crecip_part<C>(L, part, zr, zi, prec, o.s, o.e, o.l);
}

// the row swaps of P, composed into one permutation (one thread: integer work only), then
// applied as a parallel gather B -> X and a parallel copy X -> B
__global__ void lu_perm_kernel(int64_t n, const int64_t *ipiv, int64_t *perm)
{
    if (threadIdx.x || blockIdx.x) return;
    for (int64_t i = 0; i < n; i++) perm[i] = i;
    for (int64_t c = 0; c < n; c++) {
        const int64_t p = ipiv[c];
        if (p != c) { const int64_t t = perm[c]; perm[c] = perm[p]; perm[p] = t; }
    }
}

// X row r := B row perm[r] (one thread per word)
__global__ void lu_gather_kernel(int L, DMatOut bre, DMatOut bim, DMatOut xre, DMatOut xim, int64_t n, int64_t nrhs,
                                 const int64_t *perm)
{
    const int64_t per = 2 * (int64_t)L;
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n * nrhs * per) return;
    const int64_t e = g / per;
    const int w = (int)(g - e * per);
    const int part = w >= L, l = w - part * L;
    const int64_t r = e / nrhs, q = e - r * nrhs, src = perm[r];
    const DMatOut &Bm = part ? bim : bre, &Xm = part ? xim : xre;
    Xm.limbs[(r * Xm.ld + q) * L + l] = Bm.limbs[(src * Bm.ld + q) * L + l];
    if (l == 0) {
        Xm.sign[r * Xm.ld + q] = Bm.sign[src * Bm.ld + q];
        Xm.exp[r * Xm.ld + q] = Bm.exp[src * Bm.ld + q];
    }
}

template <int C>
__global__ void __launch_bounds__(128) lu_fwd_kernel(int L, DMatOut fre, DMatOut fim, DMatOut bre, DMatOut bim,
                                                     int64_t c, int64_t n, int64_t nrhs, int prec)
{
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int part = (int)(g & 1);
    const int64_t x = g >> 1;
    if (x >= (n - c - 1) * nrhs) return;
    const int64_t r = c + 1 + x / nrhs, q = x % nrhs;
    const Num<C> lr = ld<C>(L, el(L, fre, r, c)), li = ld<C>(L, el(L, fim, r, c));
    const Num<C> yr = ld<C>(L, el(L, bre, c, q)), yi = ld<C>(L, el(L, bim, c, q));
    const El a = el(L, part ? bim : bre, r, q);
    const Num<C> av = ld<C>(L, a);
    cfms_part<C>(L, part, &av, lr, li, yr, yi, prec, a.s, a.e, a.l);
}

// x = cmul(B_cq, 1/U_cc): each lane of the pair computes one part and they swap parts by shuffle
template <int C>
__global__ void __launch_bounds__(128) lu_bwd_kernel(int L, DMatOut fre, DMatOut fim, DMatOut bre, DMatOut bim,
                                                     DMatOut xre, DMatOut xim, DMatOut rre, DMatOut rim,
                                                     int64_t c, int64_t nrhs, int prec)
{
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int part = (int)(g & 1);
    const int64_t x = g >> 1;
    if (x >= (c + 1) * nrhs) return;                   // pairs leave together
    const unsigned pm = 3u << (threadIdx.x & 30);
    const int64_t r = x / nrhs, q = x % nrhs;
    const Num<C> yr = ld<C>(L, el(L, bre, c, q)), yi = ld<C>(L, el(L, bim, c, q));
    const Num<C> wr = ld<C>(L, el(L, rre, 0, c)), wi = ld<C>(L, el(L, rim, 0, c));
    uint8_t s2[2]; int64_t e2[2]; uint64_t l2[2][C];
    cfms_part<C>(L, part, nullptr, yr, yi, wr, wi, prec, &s2[part], &e2[part], l2[part]);
    // exchange: the other part arrives from the partner lane
    const int o = part ^ 1;
    s2[o] = (uint8_t)__shfl_xor_sync(pm, (int)s2[part], 1);
    e2[o] = __shfl_xor_sync(pm, e2[part], 1);
#pragma unroll
    for (int w = 0; w < C; w++) {
        const uint64_t mine = w < L ? l2[part][w] : 0ull;
        const uint64_t other = __shfl_xor_sync(pm, mine, 1);
        if (w < L) l2[o][w] = other;
    }
    if (r == c) {
        put_part(el(L, part ? xim : xre, c, q), s2[part], e2[part], l2[part], L);
        return;
    }
    const Num<C> vr = load<C>(L, &s2[0], &e2[0], l2[0]), vi = load<C>(L, &s2[1], &e2[1], l2[1]);
    const Num<C> ur = ld<C>(L, el(L, fre, r, c)), ui = ld<C>(L, el(L, fim, r, c));
    const El a = el(L, part ? bim : bre, r, q);
    const Num<C> av = ld<C>(L, a);
    cfms_part<C>(L, part, &av, ur, ui, vr, vi, prec, a.s, a.e, a.l);
}

__global__ void lu_copy_kernel(int L, DMatOut xre, DMatOut xim, DMatOut bre, DMatOut bim, int64_t n, int64_t nrhs)
{
    const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= n * nrhs) return;
    const int64_t r = x / nrhs, q = x % nrhs;
    for (int part = 0; part < 2; part++) {
        const El s_ = el(L, part ? xim : xre, r, q), d = el(L, part ? bim : bre, r, q);
        *d.s = *s_.s; *d.e = *s_.e;
        for (int w = 0; w < L; w++) d.l[w] = s_.l[w];
    }
}

// ---------------------------------------------------------------- elementwise (tests)
// op 0: O = X Y ; 1: O = A - X Y ; 2: O = 1 / X ; 3: key of X -> kv[2t] = e, kv[2t+1] = v bits
template <int C>
__global__ void mp_scalar_kernel(int L, int op, int64_t cnt, int prec, DMatOut Ar, DMatOut Ai, DMatOut Xr, DMatOut Xi,
                                 DMatOut Yr, DMatOut Yi, DMatOut Or, DMatOut Oi, int64_t *kv)
{
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int part = (int)(g & 1);
    const int64_t t = g >> 1;
    if (t >= cnt) return;
    const El xr = el(L, Xr, 0, t), xi = el(L, Xi, 0, t);
    if (op == 3) {
        if (part) return;
        const Key k = pivot_key(xr.s, xr.e, xr.l, xi.s, xi.e, xi.l, L);
        kv[2 * t] = k.e;
        kv[2 * t + 1] = __double_as_longlong(k.v);
        return;
    }
    const El o = el(L, part ? Oi : Or, 0, t);
    const Num<C> x1 = ld<C>(L, xr), x2 = ld<C>(L, xi);
    if (op == 2) { crecip_part<C>(L, part, x1, x2, prec, o.s, o.e, o.l); return; }
    const Num<C> y1 = ld<C>(L, el(L, Yr, 0, t)), y2 = ld<C>(L, el(L, Yi, 0, t));
    if (op == 0) { cfms_part<C>(L, part, nullptr, x1, x2, y1, y2, prec, o.s, o.e, o.l); return; }
    const Num<C> av = ld<C>(L, el(L, part ? Ai : Ar, 0, t));
    cfms_part<C>(L, part, &av, x1, x2, y1, y2, prec, o.s, o.e, o.l);
}

// 1 / A_cc into the scratch, one warp per part (L <= 12); *info = c + 1 on the first zero pivot
__global__ void __launch_bounds__(64) lu_recip_wkernel(int L, DMatOut re, DMatOut im, int64_t c, int prec, uint8_t *rs,
                                                       int64_t *rexp, uint64_t *rl, int32_t *info)
{
    const int lane = threadIdx.x & 31, part = threadIdx.x >> 5;
    const mpw::WNum zr = wld(L, re, c, c, lane), zi = wld(L, im, c, c, lane);
    if (zr.zero && zi.zero) {
        if (part == 0 && lane == 0 && info && *info == 0) *info = (int32_t)(c + 1);
        if (lane == 0) { rs[part] = 0; rexp[part] = 0; }
        if (lane < L) rl[part * L + lane] = 0;
        return;
    }
    mpw::crecip_warp(L, part, zr, zi, prec, rs + part, rexp + part, rl + part * L, lane);
}

// recip + scale in one launch (L <= 12, few rows): warps 0 and 1 of every block compute the two
// parts of 1 / A_cc into shared memory (block 0 also stores them and the zero-pivot flag), then
// every warp scales its element part: A_rc := cmul(A_rc, 1 / A_cc), r in [r0, r1)
__global__ void __launch_bounds__(256) lu_recip_scale_wkernel(int L, DMatOut re, DMatOut im, int64_t r0, int64_t r1,
                                                              int64_t c, int prec, uint8_t *rs, int64_t *rexp,
                                                              uint64_t *rl, int32_t *info)
{
    __shared__ uint8_t ss[2];
    __shared__ int64_t se[2];
    __shared__ uint64_t sl[2][16];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, part = warp & 1;
    if (warp < 2) {
        const mpw::WNum zr = wld(L, re, c, c, lane), zi = wld(L, im, c, c, lane);
        if (zr.zero && zi.zero) {
            if (blockIdx.x == 0 && part == 0 && lane == 0 && info && *info == 0) *info = (int32_t)(c + 1);
            if (lane == 0) { ss[part] = 0; se[part] = 0; }
            if (lane < L) sl[part][lane] = 0;
        } else {
            mpw::crecip_warp(L, part, zr, zi, prec, &ss[part], &se[part], sl[part], lane);
        }
    }
    const int64_t r = r0 + (int64_t)blockIdx.x * 4 + (warp >> 1);
    const bool on = r < r1;
    mpw::WNum xr{}, xi{};
    if (on) { xr = wld(L, re, r, c, lane); xi = wld(L, im, r, c, lane); }
    __syncthreads();                                  // recip in shared memory; operands in registers
    if (blockIdx.x == 0 && warp < 2) {
        if (lane < L) rl[part * L + lane] = sl[part][lane];
        if (lane == 0) { rs[part] = ss[part]; rexp[part] = se[part]; }
    }
    if (!on) return;
    const mpw::WNum yr = mpw::wload(L, &ss[0], &se[0], sl[0], lane), yi = mpw::wload(L, &ss[1], &se[1], sl[1], lane);
    const El o = el(L, part ? im : re, r, c);
    mpw::cfms_warp(L, part, false, xr, xr, xi, yr, yi, prec, o.s, o.e, o.l, lane);
}

// Eq. 7 solve steps, warp-cooperative (L <= 12): forward B_rq := cfms(B_rq, L_rc, B_cq), one
// warp per (r, q, part)
__global__ void __launch_bounds__(256) lu_fwd_wkernel(int L, DMatOut fre, DMatOut fim, DMatOut bre, DMatOut bim,
                                                      int64_t c, int64_t n, int64_t nrhs, int prec)
{
    const int lane = threadIdx.x & 31;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int part = (int)(w & 1);
    const int64_t x = w >> 1;
    if (x >= (n - c - 1) * nrhs) return;
    const int64_t r = c + 1 + x / nrhs, q = x % nrhs;
    const mpw::WNum lr = wld(L, fre, r, c, lane), li = wld(L, fim, r, c, lane);
    const mpw::WNum yr = wld(L, bre, c, q, lane), yi = wld(L, bim, c, q, lane);
    const El a = el(L, part ? bim : bre, r, q);
    const mpw::WNum av = mpw::wload(L, a.s, a.e, a.l, lane);
    __syncwarp();
    mpw::cfms_warp(L, part, true, av, lr, li, yr, yi, prec, a.s, a.e, a.l, lane);
}

// backward: x = cmul(B_cq, 1/U_cc) -- the two warps of an element's pair compute one part each
// into shared memory -- then B_rq := cfms(B_rq, U_rc, x) (r < c) or X_cq := x (r == c)
__global__ void __launch_bounds__(256) lu_bwd_wkernel(int L, DMatOut fre, DMatOut fim, DMatOut bre, DMatOut bim,
                                                      DMatOut xre, DMatOut xim, DMatOut rre, DMatOut rim,
                                                      int64_t c, int64_t nrhs, int prec)
{
    __shared__ uint8_t ss[4][2];
    __shared__ int64_t se[4][2];
    __shared__ uint64_t sl[4][2][16];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, part = warp & 1, slot = warp >> 1;
    const int64_t x = (int64_t)blockIdx.x * 4 + slot;
    const bool on = x < (c + 1) * nrhs;
    const int64_t r = on ? x / nrhs : 0, q = on ? x % nrhs : 0;
    if (on) {
        const mpw::WNum yr = wld(L, bre, c, q, lane), yi = wld(L, bim, c, q, lane);
        const mpw::WNum wr = wld(L, rre, 0, c, lane), wi = wld(L, rim, 0, c, lane);
        mpw::cfms_warp(L, part, false, yr, yr, yi, wr, wi, prec, &ss[slot][part], &se[slot][part], sl[slot][part], lane);
    }
    __syncthreads();
    if (!on) return;
    if (r == c) {
        const El o = el(L, part ? xim : xre, c, q);
        if (lane < L) o.l[lane] = sl[slot][part][lane];
        if (lane == 0) { *o.s = ss[slot][part]; *o.e = se[slot][part]; }
        return;
    }
    const mpw::WNum vr = mpw::wload(L, &ss[slot][0], &se[slot][0], sl[slot][0], lane);
    const mpw::WNum vi = mpw::wload(L, &ss[slot][1], &se[slot][1], sl[slot][1], lane);
    const mpw::WNum ur = wld(L, fre, r, c, lane), ui = wld(L, fim, r, c, lane);
    const El a = el(L, part ? bim : bre, r, q);
    const mpw::WNum av = mpw::wload(L, a.s, a.e, a.l, lane);
    __syncwarp();
    mpw::cfms_warp(L, part, true, av, ur, ui, vr, vi, prec, a.s, a.e, a.l, lane);
}

// op 0 / 1 of mp_scalar_kernel, warp-cooperative (L <= 12)
__global__ void __launch_bounds__(256) mp_scalar_wkernel(int L, int op, int64_t cnt, int prec, DMatOut Ar, DMatOut Ai,
                                                         DMatOut Xr, DMatOut Xi, DMatOut Yr, DMatOut Yi, DMatOut Or,
                                                         DMatOut Oi)
{
    const int lane = threadIdx.x & 31;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int part = (int)(w & 1);
    const int64_t t = w >> 1;
    if (t >= cnt) return;
    const mpw::WNum x1 = wld(L, Xr, 0, t, lane), x2 = wld(L, Xi, 0, t, lane);
    const El o = el(L, part ? Oi : Or, 0, t);
    if (op == 2) {
        if (x1.zero && x2.zero) {                      // (the tests pass nonzero z only)
            if (lane < L) o.l[lane] = 0;
            if (lane == 0) { *o.s = 0; *o.e = 0; }
            return;
        }
        mpw::crecip_warp(L, part, x1, x2, prec, o.s, o.e, o.l, lane);
        return;
    }
    const mpw::WNum y1 = wld(L, Yr, 0, t, lane), y2 = wld(L, Yi, 0, t, lane);
    const mpw::WNum av = op == 1 ? wld(L, part ? Ai : Ar, 0, t, lane) : x1;
    mpw::cfms_warp(L, part, op == 1, av, x1, x2, y1, y2, prec, o.s, o.e, o.l, lane);
}

// ---------------------------------------------------------------- launchers (L dispatch)
// Warp kernels (L <= 12) run a launch when it has at most MPCGEMM_MPWARP_MAX elements (default
// 1024 for L <= 8, 4096 above, where the thread-per-part code is slower; 0: never): a warp per
// element part issues ~32x the instructions of a thread per part, so it pays only while the
// launch is latency-bound (few elements)
static int64_t mpw_max(int L) {
    const char *e = getenv("MPCGEMM_MPWARP_MAX");
    return e && *e ? atoll(e) : (L > 8 ? 4096 : 1024);
}

// capacity instantiation for L limbs: 4, 8 or 16
#define MPC_DISPATCH_C(L, KERNEL_CALL)                        \
    do {                                                      \
        if ((L) <= 4) { constexpr int C = 4; KERNEL_CALL; }   \
        else if ((L) <= 8) { constexpr int C = 8; KERNEL_CALL; } \
        else if ((L) <= 12) { constexpr int C = 12; KERNEL_CALL; } \
        else { constexpr int C = 16; KERNEL_CALL; }           \
    } while (0)

cudaError_t lu_pivot_launch(int L, DMatOut re, DMatOut im, int64_t n, int64_t c, int64_t *ipiv, cudaStream_t st) {
    if (L < 1 || L > mps::kLMax) return cudaErrorInvalidValue;
    lu_pivot_kernel<<<1, 1024, 0, st>>>(L, re, im, n, c, ipiv);
    return cudaGetLastError();
}

cudaError_t lu_swap_launch(int L, DMatOut re, DMatOut im, int64_t ncols, int64_t c, const int64_t *ipiv, cudaStream_t st) {
    const unsigned g = (unsigned)((ncols * 2 * L + 255) / 256);
    if (L < 1 || L > mps::kLMax) return cudaErrorInvalidValue;
    lu_swap_kernel<<<g, 256, 0, st>>>(L, re, im, ncols, c, ipiv);
    return cudaGetLastError();
}

cudaError_t lu_recip_launch(int L, DMatOut re, DMatOut im, int64_t c, int prec, LuScratch s, int32_t *info,
                            cudaStream_t st) {
    if (L < 1 || L > mps::kLMax) return cudaErrorInvalidValue;
    if (L <= 12 && mpw_max(L) > 0) {
        lu_recip_wkernel<<<1, 64, 0, st>>>(L, re, im, c, prec, s.sign, s.exp, s.limbs, info);
        return cudaGetLastError();
    }
    MPC_DISPATCH_C(L, (lu_recip_kernel<C><<<1, 2, 0, st>>>(L, re, im, c, prec, s.sign, s.exp, s.limbs, info)));
    return cudaGetLastError();
}

cudaError_t lu_recip_scale_launch(int L, DMatOut re, DMatOut im, int64_t r0, int64_t r1, int64_t c, int prec,
                                  LuScratch s, int32_t *info, int *nlaunch, cudaStream_t st) {
    if (L < 1 || L > mps::kLMax) return cudaErrorInvalidValue;
    *nlaunch = 1;
    if (L <= 12 && r1 > r0 && r1 - r0 <= mpw_max(L)) {
        lu_recip_scale_wkernel<<<(unsigned)((r1 - r0 + 3) / 4), 256, 0, st>>>(L, re, im, r0, r1, c, prec, s.sign, s.exp,
                                                                              s.limbs, info);
        return cudaGetLastError();
    }
    cudaError_t e = lu_recip_launch(L, re, im, c, prec, s, info, st);
    if (e != cudaSuccess) return e;
    *nlaunch = r1 > r0 ? 2 : 1;
    return lu_scale_launch(L, re, im, r0, r1, c, prec, s, st);
}

cudaError_t lu_scale_launch(int L, DMatOut re, DMatOut im, int64_t r0, int64_t r1, int64_t c, int prec, LuScratch s,
                            cudaStream_t st) {
    if (r1 <= r0) return cudaSuccess;
    const unsigned g = (unsigned)((2 * (r1 - r0) + 127) / 128);
    if (L < 1 || L > mps::kLMax) return cudaErrorInvalidValue;
    if (L <= 12 && r1 - r0 <= mpw_max(L)) {
        lu_scale_wkernel<<<(unsigned)((r1 - r0 + 3) / 4), 256, 0, st>>>(L, re, im, r0, r1, c, prec, s.sign, s.exp, s.limbs);
        return cudaGetLastError();
    }
    MPC_DISPATCH_C(L, (lu_scale_kernel<C><<<g, 128, 0, st>>>(L, re, im, r0, r1, c, prec, s.sign, s.exp, s.limbs)));
    return cudaGetLastError();
}

cudaError_t lu_update_launch(int L, DMatOut re, DMatOut im, int64_t r0, int64_t r1, int64_t t0, int64_t t1, int64_t c,
                             int prec, cudaStream_t st) {
    if (r1 <= r0 || t1 <= t0) return cudaSuccess;
    if (L >= 1 && L <= 12 && (r1 - r0) * (t1 - t0) <= mpw_max(L)) {
        const int64_t warps = (r1 - r0) * (t1 - t0) * 2;
        const int64_t blocks = std::min<int64_t>((warps + 7) / 8, 148 * 64);
        lu_update_wkernel<<<(unsigned)blocks, 256, 0, st>>>(L, re, im, r0, r1, t0, t1, c, prec);
        return cudaGetLastError();
    }
    const int64_t rows = r1 - r0;
    const int64_t gx = (2 * (t1 - t0) + 127) / 128;
    int64_t gy = rows;
    const int64_t want = 148 * 16;                            // ~16 CTAs of 128 threads per SM
    if (gx * gy > want) gy = (want + gx - 1) / gx;
    if (gy < 1) gy = 1;
    if (gy > 65535) gy = 65535;
    dim3 grid((unsigned)gx, (unsigned)gy);
    if (L < 1 || L > mps::kLMax) return cudaErrorInvalidValue;
    MPC_DISPATCH_C(L, (lu_update_kernel<C><<<grid, 128, 0, st>>>(L, re, im, r0, r1, t0, t1, c, prec)));
    return cudaGetLastError();
}

cudaError_t lu_solve_launch(int L, DMatOut fre, DMatOut fim, int64_t n, const int64_t *ipiv, DMatOut bre, DMatOut bim,
                            int64_t nrhs, int prec, SolveScratch s, cudaStream_t st) {
    if (L < 1 || L > mps::kLMax) return cudaErrorInvalidValue;
    MPC_DISPATCH_C(L, (lu_recip_all_kernel<C><<<(unsigned)((2 * n + 127) / 128), 128, 0, st>>>(L, fre, fim, n, prec, s.rre, s.rim)));
    lu_perm_kernel<<<1, 1, 0, st>>>(n, ipiv, s.perm);
    lu_gather_kernel<<<(unsigned)((n * nrhs * 2 * L + 255) / 256), 256, 0, st>>>(L, bre, bim, s.xre, s.xim, n, nrhs, s.perm);
    lu_copy_kernel<<<(unsigned)((n * nrhs + 127) / 128), 128, 0, st>>>(L, s.xre, s.xim, bre, bim, n, nrhs);
    const int64_t wmax = mpw_max(L);
    for (int64_t c = 0; c + 1 < n; c++) {
        if (L <= 12 && (n - c - 1) * nrhs <= wmax)
            lu_fwd_wkernel<<<(unsigned)(((n - c - 1) * nrhs * 2 + 7) / 8), 256, 0, st>>>(L, fre, fim, bre, bim, c, n, nrhs, prec);
        else
            MPC_DISPATCH_C(L, (lu_fwd_kernel<C><<<(unsigned)((2 * (n - c - 1) * nrhs + 127) / 128), 128, 0, st>>>(L, fre, fim, bre, bim, c, n, nrhs, prec)));
    }
    for (int64_t c = n - 1; c >= 0; c--) {
        if (L <= 12 && (c + 1) * nrhs <= wmax)
            lu_bwd_wkernel<<<(unsigned)(((c + 1) * nrhs + 3) / 4), 256, 0, st>>>(L, fre, fim, bre, bim, s.xre, s.xim, s.rre, s.rim,
                                                                                   c, nrhs, prec);
        else
            MPC_DISPATCH_C(L, (lu_bwd_kernel<C><<<(unsigned)((2 * (c + 1) * nrhs + 127) / 128), 128, 0, st>>>(L, fre, fim, bre, bim, s.xre, s.xim,
                                                                                 s.rre, s.rim, c, nrhs, prec)));
    }
    lu_copy_kernel<<<(unsigned)((n * nrhs + 127) / 128), 128, 0, st>>>(L, s.xre, s.xim, bre, bim, n, nrhs);
    return cudaGetLastError();
}

cudaError_t mp_scalar_launch(int L, int op, int64_t cnt, int prec, DMatOut Ar, DMatOut Ai, DMatOut Xr, DMatOut Xi,
                             DMatOut Yr, DMatOut Yi, DMatOut Or, DMatOut Oi, int64_t *kv, cudaStream_t st) {
    if (cnt <= 0) return cudaSuccess;
    const unsigned g = (unsigned)((2 * cnt + 127) / 128);
    if (L < 1 || L > mps::kLMax) return cudaErrorInvalidValue;
    if ((op == 0 || op == 1 || op == 2) && L <= 12 && mpw_max(L) > 0) {
        mp_scalar_wkernel<<<(unsigned)((2 * cnt + 7) / 8), 256, 0, st>>>(L, op, cnt, prec, Ar, Ai, Xr, Xi, Yr, Yi, Or, Oi);
        return cudaGetLastError();
    }
    MPC_DISPATCH_C(L, (mp_scalar_kernel<C><<<g, 128, 0, st>>>(L, op, cnt, prec, Ar, Ai, Xr, Xi, Yr, Yi, Or, Oi, kv)));
    return cudaGetLastError();
}

}  // namespace mpc
