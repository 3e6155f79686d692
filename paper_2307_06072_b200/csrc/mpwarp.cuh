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

}  // namespace mpw
}  // namespace mpc
