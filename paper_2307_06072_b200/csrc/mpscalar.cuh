// mpscalar.cuh -- per-thread multiple-precision scalar arithmetic for the NEXT-3 complex LU
// (PAPER.md:243-263).  MPC-style semantics: every real part of a complex
// result is the EXACT value rounded once to prec (round to nearest, ties to even):
//   cmul(x, y)    = ( RNE(xr yr - xi yi), RNE(xr yi + xi yr) )
//   cfms(a, x, y) = ( RNE(ar - (xr yr - xi yi)), RNE(ai - (xr yi + xi yr)) )
//   crecip(z)     = ( RNE(zr / (zr^2 + zi^2)), RNE(-zi / (zr^2 + zi^2)) )
// Exact sums of up to three signed terms are formed cluster by cluster (a term joins the
// current cluster if its top bit lies above the cluster's lowest bit minus prec + 4); terms
// below a nonzero cluster sum only decide the direction of a sticky unit placed under the
// rounding position, which reproduces the rounding of the exact sum (DESIGN.md NEXT-3).
// Element format: the ABI's (include/mpcgemm.h) -- value = (-1)^sign N 2^(exp - 64 L).
#pragma once
#include <cstdint>
#include "common.cuh"

namespace mpc {
namespace mps {

MPC_DEV int bitlen(const uint64_t *p, int n) {
    for (int i = n - 1; i >= 0; i--)
        if (p[i]) return 64 * i + 64 - __clzll((long long)p[i]);
    return 0;
}

// r[0..na+nb) = a * b
MPC_DEV void mulmag(uint64_t *r, const uint64_t *a, int na, const uint64_t *b, int nb) {
    for (int i = 0; i < na + nb; i++) r[i] = 0;
    for (int i = 0; i < na; i++) {
        uint64_t carry = 0;
        const uint64_t ai = a[i];
        for (int j = 0; j < nb; j++) {
            const uint64_t lo = ai * b[j], hi = __umul64hi(ai, b[j]);
            uint64_t t = r[i + j] + lo;
            uint64_t c1 = t < lo;
            uint64_t t2 = t + carry;
            c1 += t2 < t;
            r[i + j] = t2;
            carry = hi + c1;
        }
        r[i + nb] = carry;
    }
}

// buf[0..nw) (two's complement) += (neg ? -1 : 1) * (p[0..np) << sh), sh >= 0
MPC_DEV void addsh(uint64_t *buf, int nw, const uint64_t *p, int np, int64_t sh, bool neg) {
    const int lo = (int)(sh >> 6), bs = (int)(sh & 63);
    uint64_t c = 0;
    int idx = lo;
    for (int i = 0; i <= np && idx < nw; i++, idx++) {
        uint64_t v = i < np ? (p[i] << bs) : 0ull;
        if (bs && i > 0) v |= p[i - 1] >> (64 - bs);
        const uint64_t x = buf[idx];
        if (!neg) { const uint64_t t = x + v; const uint64_t t2 = t + c; c = (t < x) + (t2 < t); buf[idx] = t2; }
        else      { const uint64_t t = x - v; const uint64_t t2 = t - c; c = (x < v) + (t < c); buf[idx] = t2; }
    }
    for (; c && idx < nw; idx++) {
        if (!neg) { buf[idx] += 1; c = buf[idx] == 0; }
        else      { c = buf[idx] == 0; buf[idx] -= 1; }
    }
}

// one exact signed term: value = (neg ? -1 : 1) * m[0..n) * 2^lsb ; top = lsb + bitlen(m)
struct Term {
    const uint64_t *m;
    int n;
    int64_t lsb, top;
    bool neg;
};

MPC_DEV Term make_term(const uint64_t *m, int n, int64_t lsb, bool neg) {
    Term t;
    t.m = m; t.n = n; t.lsb = lsb; t.neg = neg;
    const int b = bitlen(m, n);
    t.top = b ? lsb + b : INT64_MIN;
    return t;
}

// RNE of the magnitude buf[0..nw) (LSB weight 2^base) to prec bits into the ABI element
// (sign neg).  buf is modified (rounding increments).
MPC_DEV void round_store(uint64_t *buf, int nw, int64_t base, bool neg, int prec, int L,
                         uint8_t *so, int64_t *eo, uint64_t *lo)
{
    const int b = bitlen(buf, nw);
    if (!b) { *so = 0; *eo = 0; for (int l = 0; l < L; l++) lo[l] = 0; return; }
    int64_t E = base + b;                       // MPFR exponent: |v| in [2^(E-1), 2^E)
    const int rpos = b - prec - 1;              // round bit position in buf
    int rbit = 0, sticky = 0;
    if (rpos >= 0) {
        rbit = (int)((buf[rpos >> 6] >> (rpos & 63)) & 1);
        for (int l = 0; l < (rpos >> 6) && !sticky; l++) sticky = buf[l] != 0;
        if (!sticky && (rpos & 63)) sticky = (buf[rpos >> 6] & ((1ull << (rpos & 63)) - 1)) != 0;
    }
    // kept bits: [b - prec, b); their lowest is bit kpos
    const int kpos = b - prec;
    auto get64 = [&](int pos) -> uint64_t {     // 64 bits of buf from bit pos (pos may be < 0)
        if (pos <= -64) return 0ull;
        if (pos < 0) return buf[0] << (-pos);
        const int li = pos >> 6, bo = pos & 63;
        const uint64_t a = li < nw ? buf[li] : 0ull;
        if (!bo) return a;
        const uint64_t h = li + 1 < nw ? buf[li + 1] : 0ull;
        return (a >> bo) | (h << (64 - bo));
    };
    const int drop = 64 * L - prec;             // zero low bits of the ABI mantissa
    const int wb = b - 64 * L;                  // window [b - 64 L, b) -> limbs
    bool up = false;
    if (rpos >= 0) {
        const int lsbit = (int)((get64(kpos) & 1ull));
        up = rbit && (sticky || lsbit);
    }
    uint64_t c = up ? (1ull << drop) : 0ull;
    bool carry_out = false;
    for (int l = 0; l < L; l++) {
        uint64_t w = get64(wb + 64 * l);
        if (l == 0 && drop) w &= ~((1ull << drop) - 1);
        const uint64_t x = w + c;
        c = x < w ? 1ull : 0ull;
        lo[l] = x;
    }
    if (c) carry_out = true;
    if (carry_out) {                            // all kept bits were ones: 2^E
        for (int l = 0; l < L - 1; l++) lo[l] = 0;
        lo[L - 1] = 1ull << 63;
        E += 1;
    }
    *so = neg ? 1 : 0;
    *eo = E;
}

// sign (-1, 0, +1) of the exact sum of terms t[i0..cnt) (at most two), sorted by top descending
MPC_DEV int sign_of_rest(const Term *t, int i0, int cnt) {
    if (i0 >= cnt) return 0;
    if (i0 + 1 == cnt || t[i0].top > t[i0 + 1].top || t[i0].neg == t[i0 + 1].neg)
        return t[i0].neg ? -1 : 1;
    // equal tops, opposite signs: compare magnitudes aligned at the top
    const Term &a = t[i0], &b = t[i0 + 1];
    const int ba = bitlen(a.m, a.n), bb = bitlen(b.m, b.n);
    for (int q = 0; q < (ba > bb ? ba : bb); q += 64) {
        auto top64 = [&](const Term &x, int bx) -> uint64_t {   // bits [bx - q - 64, bx - q)
            const int pos = bx - q - 64;
            if (pos <= -64) return 0ull;
            if (pos < 0) return x.m[0] << (-pos);
            const int li = pos >> 6, bo = pos & 63;
            const uint64_t lo = x.m[li];
            if (!bo) return lo;
            const uint64_t hi = li + 1 < x.n ? x.m[li + 1] : 0ull;
            return (lo >> bo) | (hi << (64 - bo));
        };
        const uint64_t x = top64(a, ba), y = top64(b, bb);
        if (x != y) return (x > y) == !a.neg ? 1 : -1;
    }
    return 0;
}

// RNE(sum of the terms) to prec bits, stored in the ABI format.  t[] is reordered.
// buf: scratch of nw_max limbs (>= 9 Lmax + 6 for terms of <= 2 Lmax limbs, prec <= 64 Lmax).
MPC_DEV void sum_round(Term *t, int cnt, int prec, int L, uint64_t *buf, int nw_max,
                       uint8_t *so, int64_t *eo, uint64_t *lo)
{
    int k = 0;                                   // drop zero terms
    for (int i = 0; i < cnt; i++) if (t[i].top != INT64_MIN) t[k++] = t[i];
    cnt = k;
    for (int i = 1; i < cnt; i++)                // sort by top descending (<= 3 terms)
        for (int j = i; j > 0 && t[j].top > t[j - 1].top; j--) { Term x = t[j]; t[j] = t[j - 1]; t[j - 1] = x; }
    int i = 0;
    while (i < cnt) {
        int64_t lowb = t[i].lsb;
        const int64_t hi = t[i].top;
        int j = i + 1;
        while (j < cnt && t[j].top > lowb - (prec + 4)) { if (t[j].lsb < lowb) lowb = t[j].lsb; j++; }
        const int64_t base = lowb - (prec + 64);
        int nw = (int)((hi + 2 - base + 63) >> 6) + 1;
        if (nw > nw_max) nw = nw_max;            // cannot happen within the stated limits
        for (int q = 0; q < nw; q++) buf[q] = 0;
        for (int q = i; q < j; q++) addsh(buf, nw, t[q].m, t[q].n, t[q].lsb - base, t[q].neg);
        bool nz = false;
        for (int q = 0; q < nw && !nz; q++) nz = buf[q] != 0;
        if (!nz) { i = j; continue; }            // the cluster cancelled: the rest decides
        const int sr = sign_of_rest(t, j, cnt);
        if (sr) { const uint64_t one = 1; addsh(buf, nw, &one, 1, 0, sr < 0); }
        const bool neg = (int64_t)buf[nw - 1] < 0;
        if (neg) { uint64_t c = 1; for (int q = 0; q < nw; q++) { const uint64_t x = ~buf[q] + c; c = c && x == 0; buf[q] = x; } }
        round_store(buf, nw, base, neg, prec, L, so, eo, lo);
        return;
    }
    *so = 0; *eo = 0;
    for (int l = 0; l < L; l++) lo[l] = 0;
}

constexpr int kLMax = 16;                        // prec <= 1024 for the LU path

// Capacity-templated element: L <= C limbs used.  The kernels are instantiated for C = 4, 8,
// 12 and 16 (lu.cu) so that operands and product accumulators stay in registers (static indices
// under unrolled loops guarded by q < L) and the per-thread stack stays small.
template <int C>
struct Num {
    uint64_t m[C];
    int64_t e;        // weight of m[0]'s bit 0: exp - 64 L
    bool neg, zero;
};

template <int C>
MPC_DEV Num<C> load(int L, const uint8_t *s, const int64_t *e, const uint64_t *l) {
    Num<C> x;
    bool nz = false;
#pragma unroll
    for (int q = 0; q < C; q++) { x.m[q] = q < L ? l[q] : 0ull; nz = nz || x.m[q]; }
    x.zero = !nz;
    x.neg = nz && *s;
    x.e = *e - 64 * (int64_t)L;
    return x;
}

// p[0..2L) = a b (product scanning: a 192-bit column accumulator in registers, one store per
// limb of p)
MPC_DEV void mul_ps(uint64_t *p, const uint64_t *a, const uint64_t *b, int L) {
    uint64_t acc0 = 0, acc1 = 0, acc2 = 0;
    for (int k = 0; k < 2 * L - 1; k++) {
        const int i0 = k - (L - 1) > 0 ? k - (L - 1) : 0, i1 = k < L - 1 ? k : L - 1;
        for (int i = i0; i <= i1; i++) {
            const uint64_t x = a[i], y = b[k - i];
            const uint64_t lo = x * y, hi = __umul64hi(x, y);
            acc0 += lo;
            const uint64_t h = hi + (acc0 < lo);          // hi <= 2^64 - 2: no overflow
            acc1 += h;
            acc2 += acc1 < h;
        }
        p[k] = acc0;
        acc0 = acc1; acc1 = acc2; acc2 = 0;
    }
    p[2 * L - 1] = acc0;
}

template <int C>
MPC_DEV Term prod_term(int L, const Num<C> &x, const Num<C> &y, bool flip, uint64_t *p) {
    Term t;
    if (x.zero || y.zero) { t.m = p; t.n = 2 * L; t.lsb = 0; t.top = INT64_MIN; t.neg = false; return t; }
    mul_ps(p, x.m, y.m, L);
    return make_term(p, 2 * L, x.e + y.e, (x.neg != y.neg) != flip);
}

template <int C>
MPC_DEV Term term_of(int L, const Num<C> &x, uint64_t *pa) {
#pragma unroll
    for (int q = 0; q < C; q++) if (q < L) pa[q] = x.m[q];
    if (x.zero) { Term t; t.m = pa; t.n = L; t.lsb = 0; t.top = INT64_MIN; t.neg = false; return t; }
    return make_term(pa, L, x.e, x.neg);
}

template <int C> struct NW { static constexpr int v = 9 * C + 6; };   // sum_round scratch limbs

// ---------------------------------------------------------------- register fast path
// For C <= 12 the (at most three) terms of cfms_part are summed exactly in a fixed window of
// W = 2C + 3 limbs (top limb: headroom for the sign) whenever every nonzero term's lowest bit
// lies inside it -- exponent gaps up to ~128 bits, the LU's usual case -- and the sum is
// rounded there.  Every array index is static (runtime shifts go through a barrel shifter), so
// the whole operation stays in registers; otherwise the general sum_round above decides.  Both
// give the same bits: the window holds the exact sum, rounded like round_store.
template <int N>
MPC_DEV void shl_bits(uint64_t (&x)[N], int b) {            // x <<= b, 0 <= b < 64
    if (!b) return;
#pragma unroll
    for (int i = N - 1; i > 0; i--) x[i] = (x[i] << b) | (x[i - 1] >> (64 - b));
    x[0] <<= b;
}
template <int N>
MPC_DEV void shl_limbs(uint64_t (&x)[N], int o) {           // x <<= 64 o, 0 <= o < 64
#pragma unroll
    for (int k = 1; k < N; k <<= 1)
        if (o & k) {
#pragma unroll
            for (int i = N - 1; i >= 0; i--) x[i] = i >= k ? x[i - k] : 0ull;
        }
}
template <int N>
MPC_DEV void shr_bits(uint64_t (&x)[N], int b) {            // x >>= b, 0 <= b < 64
    if (!b) return;
#pragma unroll
    for (int i = 0; i < N - 1; i++) x[i] = (x[i] >> b) | (x[i + 1] << (64 - b));
    x[N - 1] >>= b;
}
template <int N>
MPC_DEV void shr_limbs(uint64_t (&x)[N], int o) {           // x >>= 64 o, 0 <= o < 64
#pragma unroll
    for (int k = 1; k < N; k <<= 1)
        if (o & k) {
#pragma unroll
            for (int i = 0; i < N; i++) x[i] = i + k < N ? x[i + k] : 0ull;
        }
}

// p[0..2C) = a b (limbs beyond L are zero in a Num, so the C x C product is the L x L one)
template <int C>
MPC_DEV void mul_reg(uint64_t (&p)[2 * C], const uint64_t (&a)[C], const uint64_t (&b)[C]) {
    uint64_t acc0 = 0, acc1 = 0, acc2 = 0;
#pragma unroll
    for (int k = 0; k < 2 * C - 1; k++) {
#pragma unroll
        for (int i = 0; i < C; i++) {
            const int j = k - i;
            if (j >= 0 && j < C) {
                const uint64_t x = a[i], y = b[j];
                const uint64_t lo = x * y, hi = __umul64hi(x, y);
                acc0 += lo;
                const uint64_t h = hi + (acc0 < lo);
                acc1 += h;
                acc2 += acc1 < h;
            }
        }
        p[k] = acc0;
        acc0 = acc1; acc1 = acc2; acc2 = 0;
    }
    p[2 * C - 1] = acc0;
}

// acc (two's complement, W limbs) += (neg ? -1 : 1) * m[0..N) * 2^sh, 0 <= sh, no bit beyond W
template <int W, int N>
MPC_DEV void win_add(uint64_t (&acc)[W], const uint64_t (&m)[N], int64_t sh, bool neg) {
    uint64_t t[W];
#pragma unroll
    for (int i = 0; i < W; i++) t[i] = i < N ? m[i] : 0ull;
    shl_bits(t, (int)(sh & 63));
    shl_limbs(t, (int)(sh >> 6));
    uint64_t c = 0;
#pragma unroll
    for (int i = 0; i < W; i++) {
        const uint64_t x = acc[i], v = t[i];
        if (!neg) { const uint64_t u = x + v, u2 = u + c; c = (u < x) + (u2 < u); acc[i] = u2; }
        else      { const uint64_t u = x - v, u2 = u - c; c = (x < v) + (u < c); acc[i] = u2; }
    }
}

// RNE of the magnitude acc * 2^base to prec bits, sign neg (round_store's rule)
template <int C, int W>
MPC_DEV void mag_round(uint64_t (&acc)[W], int64_t base, bool neg, int prec, int L, uint8_t *so, int64_t *eo,
                       uint64_t *lo) {
    int B = 0;
#pragma unroll
    for (int i = 0; i < W; i++) if (acc[i]) B = 64 * i + 64 - __clzll((long long)acc[i]);
    if (!B) {
        *so = 0; *eo = 0;
#pragma unroll
        for (int l = 0; l < C; l++) if (l < L) lo[l] = 0;
        return;
    }
    int64_t E = base + B;
    const int rpos = B - prec - 1;
    int rbit = 0;
    bool sticky = false;
    if (rpos >= 0) {
        const int ri = rpos >> 6, rb = rpos & 63;
#pragma unroll
        for (int i = 0; i < W; i++) {
            if (i == ri) { rbit = (int)((acc[i] >> rb) & 1); sticky = sticky || (acc[i] & ((1ull << rb) - 1)) != 0; }
            if (i < ri) sticky = sticky || acc[i] != 0;
        }
    }
    const int wb = B - 64 * L;                                // acc bits [wb, B) -> the L limbs
    if (wb >= 0) { shr_bits(acc, wb & 63); shr_limbs(acc, wb >> 6); }
    else         { shl_bits(acc, (-wb) & 63); shl_limbs(acc, (-wb) >> 6); }
    const int drop = 64 * L - prec;
    if (drop) acc[0] &= ~((1ull << drop) - 1);
    const bool up = rpos >= 0 && rbit && (sticky || ((acc[0] >> drop) & 1));
    uint64_t c = up ? (1ull << drop) : 0ull;
#pragma unroll
    for (int l = 0; l < C; l++)
        if (l < L) { const uint64_t x = acc[l] + c; c = x < acc[l]; acc[l] = x; }
    if (c) {                                                  // all kept bits were ones: 2^E
#pragma unroll
        for (int l = 0; l < C; l++) if (l < L) acc[l] = l == L - 1 ? 1ull << 63 : 0ull;
        E += 1;
    }
    *so = neg ? 1 : 0;
    *eo = E;
#pragma unroll
    for (int l = 0; l < C; l++) if (l < L) lo[l] = acc[l];
}

// RNE of the window's two's-complement value acc * 2^base to prec bits
template <int C, int W>
MPC_DEV void win_round(uint64_t (&acc)[W], int64_t base, int prec, int L, uint8_t *so, int64_t *eo, uint64_t *lo) {
    const bool neg = (int64_t)acc[W - 1] < 0;
    if (neg) {
        uint64_t c = 1;
#pragma unroll
        for (int i = 0; i < W; i++) { const uint64_t x = ~acc[i] + c; c = c && x == 0; acc[i] = x; }
    }
    mag_round<C>(acc, base, neg, prec, L, so, eo, lo);
}

// the fast path of cfms_part; false: a term lies outside the window (the caller falls back)
template <int C>
MPC_DEV bool cfms_fast(int L, int part, const Num<C> *a, const Num<C> &xr, const Num<C> &xi,
                       const Num<C> &yr, const Num<C> &yi, int prec, uint8_t *so, int64_t *eo, uint64_t *lo)
{
    constexpr int W = 2 * C + 3;
    const bool sub = a != nullptr;
    const Num<C> &v0 = part ? yi : yr, &v1 = part ? yr : yi;
    const bool z0 = xr.zero || v0.zero, z1 = xi.zero || v1.zero, za = !sub || a->zero;
    const int64_t e0 = xr.e + v0.e, e1 = xi.e + v1.e;
    int64_t H = INT64_MIN;
    if (!z0) H = e0 + 128 * L;
    if (!z1 && e1 + 128 * L > H) H = e1 + 128 * L;
    if (!za && a->e + 64 * L > H) H = a->e + 64 * L;
    if (H == INT64_MIN) {                                     // every term is zero
        *so = 0; *eo = 0;
#pragma unroll
        for (int l = 0; l < C; l++) if (l < L) lo[l] = 0;
        return true;
    }
    const int64_t base = H - 64 * (W - 1);
    if ((!z0 && e0 < base) || (!z1 && e1 < base) || (!za && a->e < base)) return false;
    uint64_t acc[W];
#pragma unroll
    for (int i = 0; i < W; i++) acc[i] = 0;
    uint64_t p[2 * C];
    // part 0: a - xr yr + xi yi (cmul: xr yr - xi yi); part 1: a - xr yi - xi yr (cmul: +, +)
    if (!z0) { mul_reg<C>(p, xr.m, v0.m); win_add(acc, p, e0 - base, (xr.neg != v0.neg) != sub); }
    if (!z1) { mul_reg<C>(p, xi.m, v1.m); win_add(acc, p, e1 - base, (xi.neg != v1.neg) != (part == 0 ? !sub : sub)); }
    if (!za) win_add(acc, a->m, a->e - base, a->neg);
    win_round<C>(acc, base, prec, L, so, eo, lo);
    return true;
}

// (operands by value: the fast path's caller keeps its copies in registers)
template <int C>
__device__ __noinline__ void cfms_general(int L, int part, bool sub, const Num<C> av, const Num<C> xr, const Num<C> xi,
                                          const Num<C> yr, const Num<C> yi, int prec, uint8_t *so, int64_t *eo,
                                          uint64_t *lo)
{
    uint64_t p1[2 * C], p2[2 * C], pa[C], buf[NW<C>::v];
    Term t[3];
    const Num<C> *a = &av;
    if (part == 0) { t[0] = prod_term<C>(L, xr, yr, sub, p1); t[1] = prod_term<C>(L, xi, yi, !sub, p2); }
    else           { t[0] = prod_term<C>(L, xr, yi, sub, p1); t[1] = prod_term<C>(L, xi, yr, sub, p2); }
    int cnt = 2;
    if (sub) t[cnt++] = term_of<C>(L, *a, pa);
    sum_round(t, cnt, prec, L, buf, NW<C>::v, so, eo, lo);
}

// one part of a - x y (a == nullptr: x y):  part 0 = re: ar - xr yr + xi yi ;
// part 1 = im: ai - xr yi - xi yr.  The kernels give each part its own thread.
template <int C>
MPC_DEV void cfms_part(int L, int part, const Num<C> *a, const Num<C> &xr, const Num<C> &xi,
                       const Num<C> &yr, const Num<C> &yi, int prec, uint8_t *so, int64_t *eo, uint64_t *lo)
{
    if constexpr (C <= 12) {
        if (cfms_fast<C>(L, part, a, xr, xi, yr, yi, prec, so, eo, lo)) return;
    }
    cfms_general<C>(L, part, a != nullptr, a ? *a : xr, xr, xi, yr, yi, prec, so, eo, lo);
}

// ---------------------------------------------------------------- division (reciprocal)
// Knuth's algorithm D on 32-bit digits: q = floor(u / v), returns remainder != 0.
// u: m + n digits (u[m+n] scratch digit appended by the caller), v: n digits, v[n-1] != 0.
MPC_DEV bool divmod32(uint32_t *u, int m, const uint32_t *vin, int n, uint32_t *q, uint32_t *vn) {
    if (n == 1) {
        uint64_t r = 0;
        for (int j = m - 1; j >= 0; j--) { const uint64_t cur = (r << 32) | u[j]; q[j] = (uint32_t)(cur / vin[0]); r = cur % vin[0]; }
        return r != 0;
    }
    const int sft = __clz(vin[n - 1]);
    for (int i = n - 1; i > 0; i--) vn[i] = (vin[i] << sft) | (sft ? (uint32_t)((uint64_t)vin[i - 1] >> (32 - sft)) : 0u);
    vn[0] = vin[0] << sft;
    u[m] = sft ? (uint32_t)((uint64_t)u[m - 1] >> (32 - sft)) : 0u;
    for (int i = m - 1; i > 0; i--) u[i] = (u[i] << sft) | (sft ? (uint32_t)((uint64_t)u[i - 1] >> (32 - sft)) : 0u);
    u[0] = u[0] << sft;
    for (int j = m - n; j >= 0; j--) {
        const uint64_t num = ((uint64_t)u[j + n] << 32) | u[j + n - 1];
        uint64_t qhat = num / vn[n - 1], rhat = num % vn[n - 1];
        while (qhat >= (1ull << 32) || qhat * vn[n - 2] > ((rhat << 32) | u[j + n - 2])) {
            qhat--; rhat += vn[n - 1];
            if (rhat >= (1ull << 32)) break;
        }
        int64_t borrow = 0;
        uint64_t carry = 0;
        for (int i = 0; i < n; i++) {
            const uint64_t p = qhat * vn[i] + carry;
            carry = p >> 32;
            const int64_t t = (int64_t)u[i + j] - (int64_t)(p & 0xFFFFFFFFull) - borrow;
            u[i + j] = (uint32_t)t;
            borrow = t < 0;
        }
        const int64_t t = (int64_t)u[j + n] - (int64_t)carry - borrow;
        u[j + n] = (uint32_t)t;
        if (t < 0) {
            qhat--;
            uint64_t c = 0;
            for (int i = 0; i < n; i++) { const uint64_t s2 = (uint64_t)u[i + j] + vn[i] + c; u[i + j] = (uint32_t)s2; c = s2 >> 32; }
            u[j + n] += (uint32_t)c;
        }
        q[j] = (uint32_t)qhat;
    }
    bool rem = false;
    for (int i = 0; i < n && !rem; i++) rem = u[i] != 0;
    return rem;
}

// RNE(num / D) to prec bits.  num = (-1)^nneg nm[0..nn) 2^ne ; D = dm[0..dn) 2^de (> 0), or, if
// drop_tail, D = dm 2^de + delta with 0 < delta below the rounding reach (see crecip).
// Scratch sizes: digits of (prec + 4 + 64 dn) + 64 bits.
template <int C>
MPC_DEV void div_round(int L, const uint64_t *nm, int nn, int64_t ne, bool nneg, const uint64_t *dm, int dn, int64_t de,
                       bool drop_tail, int prec, uint8_t *so, int64_t *eo, uint64_t *lo)
{
    constexpr int DMAX = 5 * C + 2;                          // D limbs
    constexpr int UMAX = 2 * (C + 2) + 2 * DMAX + 4;         // dividend 32-bit digits
    const int bn = bitlen(nm, nn);
    if (!bn) { *so = 0; *eo = 0; for (int l = 0; l < L; l++) lo[l] = 0; return; }
    const int bd = bitlen(dm, dn);
    int64_t sh = (int64_t)prec + 2 + bd - bn;                // q >= 2^(prec+1)
    if (sh < 0) sh = 0;
    uint32_t u[UMAX + 1], v[2 * DMAX], vn[2 * DMAX], q[UMAX];
    const int ubits = bn + (int)sh;
    const int m = (ubits + 31) / 32 + 1;
    for (int i = 0; i <= m && i <= UMAX; i++) u[i] = 0;
    // u = nm << sh
    for (int i = 0; i < nn; i++) {
        for (int h = 0; h < 2; h++) {
            const uint64_t d = (nm[i] >> (32 * h)) & 0xFFFFFFFFull;
            if (!d) continue;
            const int64_t pos = 64 * (int64_t)i + 32 * h + sh;      // bit position of digit d
            const int di = (int)(pos >> 5), bo = (int)(pos & 31);
            const uint64_t w = d << bo;
            u[di] |= (uint32_t)w;
            if (w >> 32) u[di + 1] |= (uint32_t)(w >> 32);
        }
    }
    int n = (bd + 31) / 32;
    for (int i = 0; i < n; i++) v[i] = (uint32_t)(dm[i >> 1] >> (32 * (i & 1)));
    for (int i = 0; i < m; i++) q[i] = 0;
    bool rem = divmod32(u, m, v, n, q, vn);
    // quotient digits q[0 .. m-n]
    const int qd = m - n + 1;
    uint64_t r[UMAX / 2 + 2];
    const int rn = (qd + 1) / 2 + 1;
    for (int i = 0; i < rn; i++) r[i] = 0;
    for (int i = 0; i < qd; i++) r[i >> 1] |= (uint64_t)q[i] << (32 * (i & 1));
    if (drop_tail && !rem) {                                 // exact quotient by the truncated D:
        uint64_t b = 1;                                      // the true one is just below it
        for (int i = 0; i < rn && b; i++) { b = r[i] == 0; r[i] -= 1; }
        rem = true;
    }
    // 2 q + sticky
    for (int i = rn - 1; i > 0; i--) r[i] = (r[i] << 1) | (r[i - 1] >> 63);
    r[0] = (r[0] << 1) | (rem ? 1ull : 0ull);
    round_store(r, rn, ne - de - sh - 1, nneg, prec, L, so, eo, lo);
}

// Register fast path of crecip_part (C <= 8): D = zr^2 + zi^2 exactly in 2C + 2 limbs (square
// exponents at most 120 bits apart, else false), normalised to its top bit; the numerator's
// mantissa N placed so that U = N 2^(32 + 64 (2C + 2)); q = floor(U / D) by Knuth's algorithm
// D on 32-bit digits with every index static (6C + 5 dividend digits, 4C + 4 divisor digits,
// 2C + 2 quotient digits: q >= 2^(64C + 31) > 2^(prec + 1)); then RNE of 2q + (remainder != 0),
// the same rounding input div_round builds.
template <int C>
MPC_DEV bool crecip_fast(int L, int part, const Num<C> &zr, const Num<C> &zi, int prec, uint8_t *so, int64_t *eo,
                         uint64_t *lo)
{
    constexpr int ND = 2 * C + 2;                             // divisor limbs
    constexpr int N = 2 * ND;                                 // divisor digits
    constexpr int MU = 6 * C + 5;                             // dividend digits
    constexpr int NQ = MU - N + 1;                            // quotient digits
    const Num<C> &num = part ? zi : zr;
    if (num.zero) { *so = 0; *eo = 0; for (int q = 0; q < L; q++) lo[q] = 0; return true; }
    const bool hr = !zr.zero, hi = !zi.zero;
    int64_t de;
    uint64_t D[ND];
#pragma unroll
    for (int i = 0; i < ND; i++) D[i] = 0;
    uint64_t sq[2 * C];
    if (hr && hi) {
        const int64_t gr = 2 * zr.e, gi = 2 * zi.e;
        de = gr < gi ? gr : gi;
        if ((gr > gi ? gr - gi : gi - gr) > 120) return false;
        mul_reg<C>(sq, zr.m, zr.m); win_add(D, sq, gr - de, false);
        mul_reg<C>(sq, zi.m, zi.m); win_add(D, sq, gi - de, false);
    } else {
        const Num<C> &z = hr ? zr : zi;
        de = 2 * z.e;
        mul_reg<C>(sq, z.m, z.m); win_add(D, sq, 0, false);
    }
    int bd = 0;
#pragma unroll
    for (int i = 0; i < ND; i++) if (D[i]) bd = 64 * i + 64 - __clzll((long long)D[i]);
    const int sd = 64 * ND - bd;                              // normalise: top bit at 64 ND - 1
    shl_bits(D, sd & 63);
    shl_limbs(D, sd >> 6);
    uint32_t v[N], u[MU + 1];
#pragma unroll
    for (int i = 0; i < N; i++) v[i] = (uint32_t)(D[i >> 1] >> (32 * (i & 1)));
    // N's mantissa (top bit at bit 64 L - 1) moved to the top of C limbs, placed at digit 4C + 5
    uint64_t nm[C];
#pragma unroll
    for (int i = 0; i < C; i++) nm[i] = num.m[i];
    shl_limbs(nm, C - L);
#pragma unroll
    for (int i = 0; i <= MU; i++) {
        const int k = i - (4 * C + 5);
        u[i] = (k >= 0 && k < 2 * C) ? (uint32_t)(nm[k >> 1] >> (32 * (k & 1))) : 0u;
    }
    uint32_t q[NQ];
    // qhat = floor(numr / v_top) from a binary64 estimate (|error| <= 2: numr < 2^64 carries 53
    // bits, qhat < 2^33), corrected exactly -- no 64-bit integer division in the loop
    const uint64_t vt = v[N - 1];
    const double rv = 1.0 / (double)vt;
#pragma unroll
    for (int j = NQ - 1; j >= 0; j--) {
        const uint64_t numr = ((uint64_t)u[j + N] << 32) | u[j + N - 1];
        uint64_t qhat = (uint64_t)((double)numr * rv);
        if (qhat) qhat -= 1;                                  // now qhat * vt <= numr (see below)
        while (qhat * vt > numr) qhat--;
        uint64_t rhat = numr - qhat * vt;
        while (rhat >= vt) { qhat++; rhat -= vt; }
        while (qhat >= (1ull << 32) || qhat * v[N - 2] > ((rhat << 32) | u[j + N - 2])) {
            qhat--; rhat += v[N - 1];
            if (rhat >= (1ull << 32)) break;
        }
        int64_t borrow = 0;
        uint64_t carry = 0;
#pragma unroll
        for (int i = 0; i < N; i++) {
            const uint64_t p = qhat * v[i] + carry;
            carry = p >> 32;
            const int64_t t = (int64_t)u[i + j] - (int64_t)(p & 0xFFFFFFFFull) - borrow;
            u[i + j] = (uint32_t)t;
            borrow = t < 0;
        }
        const int64_t t = (int64_t)u[j + N] - (int64_t)carry - borrow;
        u[j + N] = (uint32_t)t;
        if (t < 0) {                                          // qhat one too large: add back
            qhat--;
            uint64_t c = 0;
#pragma unroll
            for (int i = 0; i < N; i++) { const uint64_t s2 = (uint64_t)u[i + j] + v[i] + c; u[i + j] = (uint32_t)s2; c = s2 >> 32; }
            u[j + N] += (uint32_t)c;
        }
        q[j] = (uint32_t)qhat;
    }
    bool rem = false;
#pragma unroll
    for (int i = 0; i < N; i++) rem = rem || u[i] != 0;
    constexpr int RW = (NQ + 1) / 2 + 1;                      // 2 q + sticky
    uint64_t r[RW];
#pragma unroll
    for (int i = 0; i < RW; i++) {
        const uint64_t lo32 = 2 * i < NQ ? q[2 * i] : 0u, hi32 = 2 * i + 1 < NQ ? q[2 * i + 1] : 0u;
        r[i] = lo32 | (hi32 << 32);
    }
    shl_bits(r, 1);
    r[0] |= rem ? 1ull : 0ull;
    // value = (U / D_norm) 2^(num.e - de - X), X = 64 (C - L) + 32 + 64 ND - sd
    const int64_t X = 64 * (int64_t)(C - L) + 32 + 64 * (int64_t)ND - sd;
    mag_round<C>(r, num.e - de - X - 1, part ? !num.neg : num.neg, prec, L, so, eo, lo);
    return true;
}

// one part of 1 / (zr + i zi) (part 0: zr / D, part 1: -zi / D), z != 0
template <int C>
__device__ __noinline__ void crecip_general(int L, int part, const Num<C> zr, const Num<C> zi, int prec,
                                            uint8_t *so, int64_t *eo, uint64_t *lo)
{
    const Num<C> &num = part ? zi : zr;
    if (num.zero) { *so = 0; *eo = 0; for (int q = 0; q < L; q++) lo[q] = 0; return; }
    const int DMAX = 5 * L + 2;
    uint64_t sr[2 * C], si[2 * C], D[5 * C + 2], na[C];
    const bool hr = !zr.zero, hi = !zi.zero;
    int64_t tr = INT64_MIN, ti = INT64_MIN;
    if (hr) { mul_ps(sr, zr.m, zr.m, L); tr = 2 * zr.e + bitlen(sr, 2 * L); }
    if (hi) { mul_ps(si, zi.m, zi.m, L); ti = 2 * zi.e + bitlen(si, 2 * L); }
    // the larger square b, the smaller s
    const bool rb = tr >= ti;
    const uint64_t *Sb = rb ? sr : si, *Ss = rb ? si : sr;
    const int64_t Eb = rb ? 2 * zr.e : 2 * zi.e, Es = rb ? 2 * zi.e : 2 * zr.e;
    const int64_t Tb = rb ? tr : ti, Ts = rb ? ti : tr;
    bool drop = false;
    int dn;
    int64_t de;
    if (Ts == INT64_MIN) {                                   // one part is zero: D = Sb exactly
        for (int q = 0; q < 2 * L; q++) D[q] = Sb[q];
        dn = 2 * L; de = Eb;
    } else if (Tb - Ts > (int64_t)prec + 128 * L + 4) {      // Ss below the quotient's reach
        for (int q = 0; q < 2 * L; q++) D[q] = Sb[q];
        dn = 2 * L; de = Eb; drop = true;
    } else {                                                 // exact D = Sb 2^Eb + Ss 2^Es
        de = Eb < Es ? Eb : Es;
        dn = (int)((Tb - de + 63) >> 6) + 1;
        if (dn > DMAX) dn = DMAX;
        for (int q = 0; q < dn; q++) D[q] = 0;
        addsh(D, dn, Sb, 2 * L, Eb - de, false);
        addsh(D, dn, Ss, 2 * L, Es - de, false);
    }
    for (int q = 0; q < L; q++) na[q] = num.m[q];
    div_round<C>(L, na, L, num.e, part ? !num.neg : num.neg, D, dn, de, drop, prec, so, eo, lo);
}

template <int C>
MPC_DEV void crecip_part(int L, int part, const Num<C> &zr, const Num<C> &zi, int prec,
                         uint8_t *so, int64_t *eo, uint64_t *lo)
{
    if constexpr (C <= 8) {                              // (C = 12: the unrolled division's code
        if (crecip_fast<C>(L, part, zr, zi, prec, so, eo, lo)) return;   // size made it slower)
    }
    crecip_general<C>(L, part, zr, zi, prec, so, eo, lo);
}

// ---------------------------------------------------------------- pivot key
// key = (e, v): e = max MPFR exponent of the nonzero parts, v = t(re) + t(im) in binary64,
// t(x) = (top 53 bits of |x|) 2^(exp(x) - e) (0 below 2^-1000), normalised into [0.5, 1)
struct Key { int64_t e; double v; };

MPC_DEV double key_part(const uint8_t *, const int64_t *ex, const uint64_t *l, int L, int64_t e) {
    const uint64_t top = l[L - 1];
    if (!top) return 0.0;
    if (*ex - e < -1000) return 0.0;
    return ldexp((double)(top >> 11), (int)(*ex - e - 53));
}

MPC_DEV Key pivot_key(const uint8_t *sr, const int64_t *er, const uint64_t *lr,
                      const uint8_t *si, const int64_t *ei, const uint64_t *li, int L) {
    const bool zr = lr[L - 1] == 0, zi = li[L - 1] == 0;
    Key k;
    if (zr && zi) { k.e = INT64_MIN; k.v = 0.0; return k; }
    int64_t e = zr ? *ei : (zi ? *er : (*er > *ei ? *er : *ei));
    const double a = key_part(sr, er, lr, L, e), b = key_part(si, ei, li, L, e);
    double s = __dadd_rn(a, b);
    if (s >= 1.0) { s = s * 0.5; e += 1; }
    k.e = e; k.v = s;
    return k;
}

MPC_DEV bool key_greater(const Key &a, const Key &b) { return a.e > b.e || (a.e == b.e && a.v > b.v); }

}  // namespace mps
}  // namespace mpc
