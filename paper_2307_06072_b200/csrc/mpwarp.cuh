// mpwarp.cuh -- warp-cooperative multiple-precision cfms / cmul for the NEXT-3 LU (L <= 12 limbs):
// the same exactly rounded results as mpscalar.cuh's cfms_part (DESIGN.md NEXT-3), one real
// part per warp, one 64-bit limb per lane.  A single thread's dependent multiply chain is the
// latency floor of mpscalar.cuh; here the product columns, the carry propagation (ballot carry
// look-ahead), the alignment shifts (shuffles) and the rounding (ballots) run across 32 lanes.
//
// Window: the exact sum of the (<= 3) terms a, +-x1 y1, +-x2 y2 in 32 limbs (lane k = limb k,
// two's complement, lane 31 = headroom), used when every nonzero term's lowest bit lies inside
// it (exponent gaps up to 64 (31 - 2L) bits: 960 at L = 8, 448 at L = 12); otherwise lane 0 runs the general single-thread
// path on gathered operands.
#pragma once
#include <cstdint>
#include "common.cuh"
#include "mpscalar.cuh"

namespace mpc {
namespace mpw {

constexpr unsigned kAll = 0xFFFFFFFFu;
constexpr int kWLimbs = 32;

struct WNum {               // this lane's limb of an element (lane >= L: 0) and the shared fields
    uint64_t m;
    int64_t e;              // weight of limb 0's bit 0: exp - 64 L
    bool neg, zero;
};

MPC_DEV WNum wload(int L, const uint8_t *s, const int64_t *e, const uint64_t *l, int lane) {
    WNum x;
    x.m = lane < L ? l[lane] : 0ull;
    x.zero = __ballot_sync(kAll, x.m != 0) == 0;
    x.neg = !x.zero && *s;
    x.e = *e - 64 * (int64_t)L;
    return x;
}

// x + y (+ cin at lane 0) across the warp: per-lane sums, carries by look-ahead on ballots
// (generate = the lane's add overflowed, propagate = its sum is all ones; exclusive)
MPC_DEV uint64_t wadd(uint64_t x, uint64_t y, bool cin, int lane) {
    const uint64_t s = x + y;
    const unsigned G = __ballot_sync(kAll, s < x), P = __ballot_sync(kAll, s == ~0ull);
    const unsigned X = (G << 1) | (cin ? 1u : 0u);
    const unsigned Cm = (X + P) ^ P;                  // carry into each lane
    return s + ((Cm >> lane) & 1u);
}
MPC_DEV uint64_t wsub(uint64_t x, uint64_t y, int lane) { return wadd(x, ~y, true, lane); }

// the warp value v shifted left by sh >= 0 bits (limbs beyond lane 31 drop)
MPC_DEV uint64_t wshl(uint64_t v, int64_t sh, int lane) {
    const int o = (int)(sh >> 6), b = (int)(sh & 63);
    const uint64_t a = __shfl_up_sync(kAll, v, o > 31 ? 31 : o);
    const uint64_t c = __shfl_up_sync(kAll, v, o + 1 > 31 ? 31 : o + 1);
    const uint64_t va = (lane >= o && o < 32) ? a : 0ull, vc = (lane >= o + 1 && o + 1 < 32) ? c : 0ull;
    return b ? (va << b) | (vc >> (64 - b)) : va;
}
// the warp value v shifted right by sh >= 0 bits
MPC_DEV uint64_t wshr(uint64_t v, int64_t sh, int lane) {
    const int o = (int)(sh >> 6), b = (int)(sh & 63);
    const uint64_t a = __shfl_down_sync(kAll, v, o > 31 ? 31 : o);
    const uint64_t c = __shfl_down_sync(kAll, v, o + 1 > 31 ? 31 : o + 1);
    const uint64_t va = (lane + o < 32 && o < 32) ? a : 0ull, vc = (lane + o + 1 < 32 && o + 1 < 32) ? c : 0ull;
    return b ? (va >> b) | (vc << (64 - b)) : va;
}

// x y as a warp value (2L limbs in lanes 0..2L-1): lane k sums column k (192 bits), then the
// column carries are added with look-ahead
MPC_DEV uint64_t wmul(uint64_t x, uint64_t y, int L, int lane) {
    uint64_t a0 = 0, a1 = 0, a2 = 0;
    for (int i = 0; i < L; i++) {
        const uint64_t xi = __shfl_sync(kAll, x, i);
        const int src = lane - i;
        const uint64_t yj = __shfl_sync(kAll, y, src < 0 ? 0 : src);
        const uint64_t v = (src >= 0 && src < L) ? yj : 0ull;
        const uint64_t lo = xi * v, hi = __umul64hi(xi, v);
        a0 += lo;
        const uint64_t h = hi + (a0 < lo);
        a1 += h;
        a2 += a1 < h;
    }
    // limb k = a0_k + a1_{k-1} + a2_{k-2} (+ carries)
    const uint64_t b1 = __shfl_up_sync(kAll, a1, 1), b2 = __shfl_up_sync(kAll, a2, 2);
    const uint64_t u1 = a0 + (lane >= 1 ? b1 : 0ull);
    uint64_t hi = u1 < a0;
    const uint64_t u2 = u1 + (lane >= 2 ? b2 : 0ull);
    hi += u2 < u1;
    const uint64_t hin = __shfl_up_sync(kAll, hi, 1);
    return wadd(u2, lane >= 1 ? hin : 0ull, false, lane);
}

// RNE of the magnitude acc 2^base to prec bits (mpscalar round_store's rule); lane l < L gets
// result limb l; returns the exponent (sign handled by the caller); zero: all limbs 0, E = 0
MPC_DEV uint64_t wround(uint64_t acc, int64_t base, int prec, int L, int lane, int64_t *E_out) {
    const unsigned nz = __ballot_sync(kAll, acc != 0);
    if (!nz) { *E_out = 0; return 0ull; }
    const int hl = 31 - __clz(nz);
    const uint64_t top = __shfl_sync(kAll, acc, hl);
    const int B = 64 * hl + 64 - __clzll((long long)top);
    int64_t E = base + B;
    const int rpos = B - prec - 1;
    int rbit = 0;
    bool sticky = false;
    if (rpos >= 0) {
        const int ri = rpos >> 6, rb = rpos & 63;
        const uint64_t wr = __shfl_sync(kAll, acc, ri);
        rbit = (int)((wr >> rb) & 1);
        sticky = (wr & ((1ull << rb) - 1)) != 0 || (nz & ((1u << ri) - 1u)) != 0;
    }
    const int wb = B - 64 * L;                        // acc bits [wb, B) -> the L limbs
    uint64_t r = wb >= 0 ? wshr(acc, wb, lane) : wshl(acc, -(int64_t)wb, lane);
    if (lane >= L) r = 0;
    const int drop = 64 * L - prec;
    if (lane == 0 && drop) r &= ~((1ull << drop) - 1);
    const uint64_t r0 = __shfl_sync(kAll, r, 0);
    const bool up = rpos >= 0 && rbit && (sticky || ((r0 >> drop) & 1));
    if (up) {
        r = wadd(r, lane == 0 ? (1ull << drop) : 0ull, false, lane);
        if (__shfl_sync(kAll, r, L)) {                // carry out of the kept bits: 2^E
            r = lane == L - 1 ? (1ull << 63) : 0ull;
            E += 1;
        }
        if (lane >= L) r = 0;
    }
    *E_out = E;
    return r;
}

// one real part of a - x y (sub) or x y:  part 0: ar - xr yr + xi yi ; part 1: ai - xr yi - xi yr.
// Writes the ABI element (so, eo, lo) from lanes 0 .. L-1.  L <= 12.  (so, eo, lo may point to
// the warp's own registers' home -- e.g. a shared-memory staging area -- or to the matrix.)
MPC_DEV void cfms_warp(int L, int part, bool sub, const WNum &a, const WNum &xr, const WNum &xi,
                       const WNum &yr, const WNum &yi, int prec, uint8_t *so, int64_t *eo, uint64_t *lo, int lane)
{
    const WNum &v0 = part ? yi : yr, &v1 = part ? yr : yi;
    const bool z0 = xr.zero || v0.zero, z1 = xi.zero || v1.zero, za = !sub || a.zero;
    const int64_t e0 = xr.e + v0.e, e1 = xi.e + v1.e;
    int64_t H = INT64_MIN;
    if (!z0) H = e0 + 128 * L;
    if (!z1 && e1 + 128 * L > H) H = e1 + 128 * L;
    if (!za && a.e + 64 * L > H) H = a.e + 64 * L;
    if (H == INT64_MIN) {                             // every term is zero
        if (lane < L) lo[lane] = 0;
        if (lane == 0) { *so = 0; *eo = 0; }
        return;
    }
    const int64_t base = H - 64 * (kWLimbs - 1);
    if ((!z0 && e0 < base) || (!z1 && e1 < base) || (!za && a.e < base)) {
        // outside the window: lane 0 runs the general path on gathered operands
        mps::Num<16> n[5];
        const WNum *src[5] = {&a, &xr, &xi, &yr, &yi};
        for (int q = 0; q < 5; q++) {
            for (int l = 0; l < 16; l++) {
                const uint64_t v = __shfl_sync(kAll, src[q]->m, l);
                n[q].m[l] = l < L ? v : 0ull;
            }
            n[q].e = src[q]->e; n[q].neg = src[q]->neg; n[q].zero = src[q]->zero;
        }
        if (lane == 0) mps::cfms_part<16>(L, part, sub ? &n[0] : nullptr, n[1], n[2], n[3], n[4], prec, so, eo, lo);
        return;
    }
    uint64_t acc = 0;
    if (!z0) {
        const uint64_t p = wmul(xr.m, v0.m, L, lane);
        const uint64_t t = wshl(p, e0 - base, lane);
        acc = ((xr.neg != v0.neg) != sub) ? wsub(acc, t, lane) : wadd(acc, t, false, lane);
    }
    if (!z1) {
        const uint64_t p = wmul(xi.m, v1.m, L, lane);
        const uint64_t t = wshl(p, e1 - base, lane);
        const bool ng = (xi.neg != v1.neg) != (part == 0 ? !sub : sub);
        acc = ng ? wsub(acc, t, lane) : wadd(acc, t, false, lane);
    }
    if (!za) {
        const uint64_t t = wshl(a.m, a.e - base, lane);
        acc = a.neg ? wsub(acc, t, lane) : wadd(acc, t, false, lane);
    }
    const bool neg = (int64_t)__shfl_sync(kAll, acc, kWLimbs - 1) < 0;
    if (neg) acc = wadd(~acc, 0ull, true, lane);
    const bool nzv = __ballot_sync(kAll, acc != 0) != 0;
    int64_t E;
    const uint64_t r = wround(acc, base, prec, L, lane, &E);
    if (lane < L) lo[lane] = r;
    if (lane == 0) { *so = (neg && nzv) ? 1 : 0; *eo = E; }
}

// ---------------------------------------------------------------- reciprocal (L <= 12)
// 128 / 64 division helpers for Knuth's algorithm D in base 2^64 (d normalised: top bit set)
MPC_DEV uint64_t invert_limb(uint64_t d) {             // floor((2^128 - 1) / d) - 2^64
    uint64_t hi = ~d, lo = ~0ull, q = 0;               // (hi:lo) = 2^128 - 1 - d 2^64, hi < d
    for (int i = 0; i < 64; i++) {                     // restoring long division, one bit a step
        const bool top = hi >> 63;
        hi = (hi << 1) | (lo >> 63);
        lo <<= 1;
        q <<= 1;
        if (top || hi >= d) { hi -= d; q |= 1; }
    }
    return q;
}
// (u1:u0) / d with u1 < d: quotient and remainder (Moller and Granlund's 2-by-1 division)
MPC_DEV uint64_t div_preinv(uint64_t u1, uint64_t u0, uint64_t d, uint64_t v, uint64_t *r_out) {
    uint64_t q0 = v * u1, q1 = __umul64hi(v, u1);
    const uint64_t t = q0 + u0;
    q1 += u1 + (t < q0);
    q0 = t;
    q1 += 1;
    uint64_t r = u0 - q1 * d;
    if (r > q0) { q1 -= 1; r += d; }
    if (r >= d) { q1 += 1; r -= d; }
    *r_out = r;
    return q1;
}

// one part of 1 / (zr + i zi): part 0 zr / D, part 1 -zi / D, D = zr^2 + zi^2 exactly (square
// exponents <= 120 bits apart, else lane 0 runs the single-thread code on gathered operands).
// Knuth's algorithm D in base 2^64 with the divisor normalised in ND = 2L + 2 lanes, the
// numerator's mantissa placed at limb ND + 1 (quotient L + 2 limbs >= prec + 2 bits), each
// quotient limb's multiply-subtract across the warp on a sliding ND + 1-limb window of the
// dividend; then RNE of 2 q + (remainder != 0).
MPC_DEV void crecip_warp(int L, int part, const WNum &zr, const WNum &zi, int prec, uint8_t *so, int64_t *eo,
                         uint64_t *lo, int lane)
{
    const WNum &num = part ? zi : zr;
    if (num.zero) {
        if (lane < L) lo[lane] = 0;
        if (lane == 0) { *so = 0; *eo = 0; }
        return;
    }
    const bool hr = !zr.zero, hi = !zi.zero;
    int64_t de;
    uint64_t D;
    if (hr && hi) {
        const int64_t gr = 2 * zr.e, gi = 2 * zi.e;
        if ((gr > gi ? gr - gi : gi - gr) > 120) {
            mps::Num<16> n[2];
            const WNum *src[2] = {&zr, &zi};
            for (int q = 0; q < 2; q++) {
                for (int l = 0; l < 16; l++) {
                    const uint64_t v = __shfl_sync(kAll, src[q]->m, l);
                    n[q].m[l] = l < L ? v : 0ull;
                }
                n[q].e = src[q]->e; n[q].neg = src[q]->neg; n[q].zero = src[q]->zero;
            }
            if (lane == 0) mps::crecip_part<16>(L, part, n[0], n[1], prec, so, eo, lo);
            return;
        }
        de = gr < gi ? gr : gi;
        const uint64_t sr = wshl(wmul(zr.m, zr.m, L, lane), gr - de, lane);
        const uint64_t si = wshl(wmul(zi.m, zi.m, L, lane), gi - de, lane);
        D = wadd(sr, si, false, lane);
    } else {
        const WNum &z = hr ? zr : zi;
        de = 2 * z.e;
        D = wmul(z.m, z.m, L, lane);
    }
    const int ND = 2 * L + 2;                           // divisor limbs
    const unsigned nzd = __ballot_sync(kAll, D != 0);
    const int hl = 31 - __clz(nzd);
    const int bd = 64 * hl + 64 - __clzll((long long)__shfl_sync(kAll, D, hl));
    const int sd = 64 * ND - bd;                        // normalise: top bit at 64 ND - 1
    const uint64_t Dn = wshl(D, sd, lane);
    const uint64_t vt = __shfl_sync(kAll, Dn, ND - 1), v2 = __shfl_sync(kAll, Dn, ND - 2);
    const uint64_t vinv = invert_limb(vt);
    // U = N 2^(64 (ND + 1)): limbs ND+1 .. ND+L, plus the zero top limb ND+L+1.  Step j touches
    // limbs j .. j+ND only, so the warp holds that window (lane l = limb j + l), moved down one
    // limb per step (the limbs entering below are U's zeros): ND + 1 <= 27 lanes for L <= 12
    const int m = L + 1;                                // quotient limbs j = m .. 0
    uint64_t u = wshl(num.m, 64 * (int64_t)(ND + 1 - m), lane);
    uint64_t q = 0;
    for (int j = m; j >= 0; j--) {
        const uint64_t ut = __shfl_sync(kAll, u, ND), un = __shfl_sync(kAll, u, ND - 1);
        const uint64_t u2 = __shfl_sync(kAll, u, ND - 2);
        uint64_t qh, rh;
        bool rover = false;
        if (ut >= vt) {                                 // (ut == vt) qhat = 2^64 - 1
            qh = ~0ull;
            rh = un + vt;
            rover = rh < un;
        } else {
            qh = div_preinv(ut, un, vt, vinv, &rh);
        }
        while (!rover) {                                // Knuth's test with the second limb
            const uint64_t plo = qh * v2, phi = __umul64hi(qh, v2);
            if (phi > rh || (phi == rh && plo > u2)) {
                qh--;
                const uint64_t r2 = rh + vt;
                rover = r2 < rh;
                rh = r2;
            } else break;
        }
        // window -= qh Dn
        const uint64_t plo = qh * Dn, phi = __umul64hi(qh, Dn);
        const uint64_t hin = __shfl_up_sync(kAll, phi, 1);
        const uint64_t qv = wadd(plo, lane >= 1 ? hin : 0ull, false, lane);   // qh Dn, ND + 1 limbs
        u = wsub(u, qv, lane);
        if ((int64_t)__shfl_sync(kAll, u, 31) < 0) {    // qhat one too large: add back
            qh--;
            u = wadd(u, Dn, false, lane);
        }
        if (lane == j) q = qh;
        if (j) {                                        // next window: limbs j-1 .. j-1+ND
            const uint64_t d = __shfl_up_sync(kAll, u, 1);
            u = lane ? d : 0ull;
        }
    }
    const bool rem = __ballot_sync(kAll, u != 0) != 0;  // the remainder: lanes 0 .. ND-1
    uint64_t r = wshl(q, 1, lane);
    if (lane == 0 && rem) r |= 1ull;
    // value = (U / Dn) 2^(num.e - de - X), X = 64 (ND + 1) - sd
    const int64_t X = 64 * (int64_t)(ND + 1) - sd;
    int64_t E;
    const uint64_t res = wround(r, num.e - de - X - 1, prec, L, lane, &E);
    if (lane < L) lo[lane] = res;
    if (lane == 0) { *so = (part ? !num.neg : num.neg) ? 1 : 0; *eo = E; }
}

}  // namespace mpw
}  // namespace mpc
