/* oracle/mpref.c -- CPU oracle for the Ozaki-scheme complex multiple-precision GEMM.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load or call this library.  It shares no
 * code, header, table or helper with the CUDA path (paper_2307_06072_b200/), and never
 * imports it.  Plain, slow, obviously-correct code: exact big integers built from
 * uint64 limbs and unsigned __int128 schoolbook products (no GMP), one rounding.
 *
 * Two oracles (DESIGN.md section "Oracle"):
 *  (1) orc_cgemm_exact  -- the plain definition C := AB (Eq. 1-2) with
 *      the complex product of Eq. 3 (4M) or Eq. 4 (3M),
 *      every sum exact, ONE round-to-nearest-even to prec_out (reading Z8).
 *      "rounded" mode: the MPC-like variant where each real GEMM (Eq. 5/6,
 *      PAPER.md:81-97) is exact then rounded, and every combination/sum is rounded.
 *  (2) orc_cgemm_ozaki  -- Algorithm 2 step by step, under the
 *      readings Z1/Z3/Z5/Z7/Z10/Z11 of DESIGN.md: per-row (per-column) exponent mu
 *      (common to Re/Im), fixed-point truncation to
 *      W = 8s-3 bits, the slices A_alpha = the s digits of the unique balanced radix-256
 *      representation (digit set [-128,127]), the triangle beta <= d-alpha+1
 *      (PAPER.md:174-177), exact accumulation (Z7) and one RNE rounding;
 *      complex forms by Eq. 5 (4M) / Eq. 6 (3M).
 *      orc_cgemm_ozaki_rows: the same with a per-row d (NEXT-4).
 *  plus the slice-count rule:
 *      t_ik = floor(max(|ReA_ik|,|ImA_ik|) 2^(7-eA_i)), u_kj likewise, T = t u,
 *      log2rho = log2((double)k) + 14.0 - log2((double)minT),
 *      s = min{ s >= 1 : 8 s >= prec - 4 + log2(c_M s) + log2rho + 0.1 }, c_4M = 3, c_3M = 4.
 *
 * Element format (MPFR convention): value = (-1)^sign * N * 2^(exp - 64 L),
 * N = little-endian limbs; zero <=> all limbs zero.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef unsigned __int128 u128;

typedef struct {
    uint8_t *sign;
    int64_t *exp;
    uint64_t *limbs;
    int64_t ld;
    int32_t L;
    int32_t pad_;
} orc_rmat;

/* ------------------------------------------------------------------ exact numbers */
/* value = (-1)^neg * mag * 2^e ; mag has n limbs (n == 0 <=> zero); own != 0 => malloc'ed */
typedef struct { int neg; int64_t e; int n; uint64_t *m; int own; } xn;

static void xn_free(xn *v) { if (v->own && v->m) free(v->m); v->m = NULL; v->n = 0; v->own = 0; }

static int is_zero_limbs(const uint64_t *p, int n) {
    for (int i = 0; i < n; i++) if (p[i]) return 0;
    return 1;
}

static xn entry_of(const orc_rmat *M, int64_t r, int64_t c) {
    int64_t idx = r * M->ld + c;
    xn v;
    v.m = M->limbs + idx * M->L;
    v.n = is_zero_limbs(v.m, M->L) ? 0 : M->L;
    v.neg = v.n ? (M->sign[idx] != 0) : 0;
    v.e = M->exp[idx] - 64 * (int64_t)M->L;
    v.own = 0;
    return v;
}

static int bitlen_limbs(const uint64_t *p, int n) {
    for (int i = n - 1; i >= 0; i--)
        if (p[i]) return 64 * i + (64 - __builtin_clzll(p[i]));
    return 0;
}

static int getbit(const uint64_t *p, int n, int64_t pos) {
    if (pos < 0 || pos >= 64 * (int64_t)n) return 0;
    return (int)((p[pos >> 6] >> (pos & 63)) & 1u);
}

/* r[0..nr) = (p >> sh) truncated to nr limbs (sh >= 0) */
static void shr_limbs(uint64_t *r, int nr, const uint64_t *p, int np, int64_t sh) {
    int64_t lo = sh >> 6; int bs = (int)(sh & 63);
    for (int i = 0; i < nr; i++) {
        int64_t a = lo + i;
        uint64_t v = 0;
        if (a < np) v = p[a] >> bs;
        if (bs && a + 1 < np) v |= p[a + 1] << (64 - bs);
        r[i] = v;
    }
}

/* r[0..nr) = (p << sh) truncated to nr limbs (sh >= 0) */
static void shl_limbs(uint64_t *r, int nr, const uint64_t *p, int np, int64_t sh) {
    int64_t lo = sh >> 6; int bs = (int)(sh & 63);
    for (int i = 0; i < nr; i++) {
        int64_t a = i - lo;           /* source limb */
        uint64_t v = 0;
        if (a >= 0 && a < np) v = p[a] << bs;
        if (bs && a - 1 >= 0 && a - 1 < np) v |= p[a - 1] >> (64 - bs);
        r[i] = v;
    }
}

/* magnitude product r[0..na+nb) = a * b (schoolbook) */
static void mulmag(uint64_t *r, const uint64_t *a, int na, const uint64_t *b, int nb) {
    memset(r, 0, sizeof(uint64_t) * (size_t)(na + nb));
    for (int i = 0; i < na; i++) {
        uint64_t carry = 0;
        for (int j = 0; j < nb; j++) {
            u128 t = (u128)a[i] * b[j] + r[i + j] + carry;
            r[i + j] = (uint64_t)t;
            carry = (uint64_t)(t >> 64);
        }
        r[i + nb] = carry;
    }
}

/* two's complement accumulator acc[0..na) += (neg ? -1 : +1) * (p << sh), sh >= 0 */
static void addsh(uint64_t *acc, int na, const uint64_t *p, int np, int64_t sh, int neg) {
    int64_t lo = sh >> 6; int bs = (int)(sh & 63);
    uint64_t c = 0;
    int64_t idx = lo;
    for (int i = 0; i <= np; i++, idx++) {
        uint64_t v = (i < np) ? (p[i] << bs) : 0;
        if (bs && i > 0) v |= p[i - 1] >> (64 - bs);
        if (idx >= na) break;
        if (!neg) {
            u128 t = (u128)acc[idx] + v + c;
            acc[idx] = (uint64_t)t; c = (uint64_t)(t >> 64);
        } else {
            u128 t = (u128)acc[idx] - v - c;
            acc[idx] = (uint64_t)t; c = (t >> 64) ? 1 : 0;
        }
    }
    for (; c && idx < na; idx++) {
        if (!neg) { acc[idx] += 1; c = (acc[idx] == 0); }
        else      { c = (acc[idx] == 0); acc[idx] -= 1; }
    }
}

/* two's complement acc (na limbs) * 2^e  ->  xn (owning) */
static xn xn_from_acc(const uint64_t *acc, int na, int64_t e) {
    xn v; v.own = 1; v.e = e;
    v.neg = (int)(acc[na - 1] >> 63);
    v.m = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(na > 0 ? na : 1));
    if (v.neg) {
        uint64_t c = 1;
        for (int i = 0; i < na; i++) { uint64_t x = ~acc[i] + c; c = (c && x == 0); v.m[i] = x; }
    } else {
        memcpy(v.m, acc, sizeof(uint64_t) * (size_t)na);
    }
    int b = bitlen_limbs(v.m, na);
    v.n = (b + 63) / 64;
    if (!v.n) v.neg = 0;
    return v;
}

/* exact a + (sub ? -b : b) */
static xn xn_add(const xn *a, const xn *b, int sub) {
    int64_t emin = 0, top = 0; int any = 0;
    const xn *t[2] = {a, b};
    for (int q = 0; q < 2; q++) {
        if (!t[q]->n) continue;
        int64_t hi = t[q]->e + 64 * (int64_t)t[q]->n;
        if (!any || t[q]->e < emin) emin = t[q]->e;
        if (!any || hi > top) top = hi;
        any = 1;
    }
    if (!any) { xn z = {0, 0, 0, NULL, 0}; return z; }
    int na = (int)((top - emin) / 64) + 3;
    uint64_t *acc = (uint64_t *)calloc((size_t)na, sizeof(uint64_t));
    if (a->n) addsh(acc, na, a->m, a->n, a->e - emin, a->neg);
    if (b->n) addsh(acc, na, b->m, b->n, b->e - emin, b->neg ^ sub);
    xn r = xn_from_acc(acc, na, emin);
    free(acc);
    return r;
}

/* RNE of v to prec bits, stored in ABI element format with Lout limbs (Z8) */
static void xn_store(const xn *v, int prec, uint8_t *sign, int64_t *exp, uint64_t *limbs, int Lout) {
    int b = v->n ? bitlen_limbs(v->m, v->n) : 0;
    memset(limbs, 0, sizeof(uint64_t) * (size_t)Lout);
    if (b == 0) { *sign = 0; *exp = 0; return; }
    int64_t E = v->e + b;
    int nq = (prec + 63) / 64 + 1;
    uint64_t q[nq];
    if (b <= prec) {
        shl_limbs(limbs, Lout, v->m, v->n, 64 * (int64_t)Lout - b);
    } else {
        int64_t sh = b - prec;
        shr_limbs(q, nq, v->m, v->n, sh);
        int rbit = getbit(v->m, v->n, sh - 1);
        int sticky = 0;                        /* OR of the bits below the round bit */
        int64_t full = (sh - 1) >> 6;
        for (int64_t q2 = 0; q2 < full && q2 < v->n && !sticky; q2++) if (v->m[q2]) sticky = 1;
        if (!sticky && full < v->n && ((sh - 1) & 63))
            if (v->m[full] & ((1ULL << ((sh - 1) & 63)) - 1)) sticky = 1;
        if (rbit && (sticky || (q[0] & 1))) {
            uint64_t c = 1;
            for (int i = 0; i < nq && c; i++) { q[i] += 1; c = (q[i] == 0); }
            if (bitlen_limbs(q, nq) > prec) {     /* carry-out: 2^prec -> 2^(prec-1), exp + 1 */
                uint64_t t2[nq];
                shr_limbs(t2, nq, q, nq, 1);
                memcpy(q, t2, sizeof(t2));
                E += 1;
            }
        }
        shl_limbs(limbs, Lout, q, nq, 64 * (int64_t)Lout - prec);
    }
    *sign = (uint8_t)v->neg;
    *exp = E;
}

/* RNE of v to prec bits as an exact number (for the MPC-like rounded mode) */
static xn xn_round(const xn *v, int prec) {
    int L = (prec + 63) / 64;
    xn r; r.own = 1; r.m = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)L);
    uint8_t s; int64_t E;
    xn_store(v, prec, &s, &E, r.m, L);
    r.n = is_zero_limbs(r.m, L) ? 0 : L;
    r.neg = r.n ? s : 0;
    r.e = E - 64 * (int64_t)L;
    return r;
}

/* exact sum_v sg[v] * sum_k X[v][k] * Y[v][k]   (Eq. 2) */
static xn dot_exact(int64_t k, int nv, xn *const *X, xn *const *Y, const int *sg) {
    int64_t emin = 0, top = 0; int any = 0, maxn = 0;
    for (int v = 0; v < nv; v++)
        for (int64_t q = 0; q < k; q++) {
            const xn *x = &X[v][q], *y = &Y[v][q];
            if (!x->n || !y->n) continue;
            int64_t lo = x->e + y->e, hi = lo + 64 * (int64_t)(x->n + y->n);
            if (!any || lo < emin) emin = lo;
            if (!any || hi > top) top = hi;
            if (x->n + y->n > maxn) maxn = x->n + y->n;
            any = 1;
        }
    if (!any) { xn z = {0, 0, 0, NULL, 0}; return z; }
    int cntbits = 2; while ((1LL << cntbits) < k * nv + 1) cntbits++;
    int na = (int)((top - emin + cntbits + 2) / 64) + 2;
    uint64_t *acc = (uint64_t *)calloc((size_t)na, sizeof(uint64_t));
    uint64_t *prod = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)maxn);
    for (int v = 0; v < nv; v++)
        for (int64_t q = 0; q < k; q++) {
            const xn *x = &X[v][q], *y = &Y[v][q];
            if (!x->n || !y->n) continue;
            mulmag(prod, x->m, x->n, y->m, y->n);
            addsh(acc, na, prod, x->n + y->n, x->e + y->e - emin, x->neg ^ y->neg ^ (sg[v] < 0));
        }
    xn r = xn_from_acc(acc, na, emin);
    free(acc); free(prod);
    return r;
}

static int nthreads_of(int32_t req) {
#ifdef _OPENMP
    return req > 0 ? req : omp_get_max_threads();
#else
    (void)req; return 1;
#endif
}

static void out_ptrs(orc_rmat *C, int64_t oi, uint8_t **s, int64_t **e, uint64_t **l) {
    *s = C->sign + oi; *e = C->exp + oi; *l = C->limbs + oi * C->L;
}

/* ------------------------------------------------------------------ oracle (1): exact */
/* form 4: Eq. 3 / Eq. 5 ; form 3: Eq. 4 / Eq. 6.
 * rounded_prec == 0 : every operation exact, one RNE to prec_out.
 * rounded_prec  > 0 : MPC-like: the 3M sums ReA+ImA, ReB+ImB, each real GEMM and every
 *                     combination are rounded to rounded_prec (then output RNE to prec_out).
 * nsamp < 0 : all m x n outputs at C[i*ld+j];  nsamp >= 0 : outputs (si[t], sj[t]) at C[t]. */
int orc_cgemm_exact(int64_t m, int64_t n, int64_t k,
                    const orc_rmat *Are, const orc_rmat *Aim, const orc_rmat *Bre, const orc_rmat *Bim,
                    orc_rmat *Cre, orc_rmat *Cim, int32_t prec_out, int32_t form, int32_t rounded_prec,
                    int64_t nsamp, const int64_t *si, const int64_t *sj, int32_t nthreads)
{
    if (m < 0 || n < 0 || k < 0 || (form != 3 && form != 4) || prec_out < 2) return -1;
    int64_t total = nsamp < 0 ? m * n : nsamp;
    int nt = nthreads_of(nthreads);
    int err = 0;
    #pragma omp parallel num_threads(nt)
    {
        xn *ar = (xn *)malloc(sizeof(xn) * (size_t)(k + 1)), *ai = (xn *)malloc(sizeof(xn) * (size_t)(k + 1));
        xn *br = (xn *)malloc(sizeof(xn) * (size_t)(k + 1)), *bi = (xn *)malloc(sizeof(xn) * (size_t)(k + 1));
        xn *as = (xn *)malloc(sizeof(xn) * (size_t)(k + 1)), *bs = (xn *)malloc(sizeof(xn) * (size_t)(k + 1));
        #pragma omp for schedule(dynamic, 1)
        for (int64_t t = 0; t < total; t++) {
            int64_t i = nsamp < 0 ? t / (n ? n : 1) : si[t];
            int64_t j = nsamp < 0 ? t % (n ? n : 1) : sj[t];
            int64_t oi = nsamp < 0 ? i * Cre->ld + j : t;
            if (i < 0 || i >= m || j < 0 || j >= n) { err = -1; continue; }
            for (int64_t q = 0; q < k; q++) {
                ar[q] = entry_of(Are, i, q); ai[q] = entry_of(Aim, i, q);
                br[q] = entry_of(Bre, q, j); bi[q] = entry_of(Bim, q, j);
            }
            xn re, im;
            if (form == 4 && !rounded_prec) {
                /* Eq. 3: Re = sum ReA ReB - ImA ImB ; Im = sum ReA ImB + ImA ReB, exact */
                xn *X1[2] = {ar, ai}, *Y1[2] = {br, bi}; int s1[2] = {+1, -1};
                xn *X2[2] = {ar, ai}, *Y2[2] = {bi, br}; int s2[2] = {+1, +1};
                re = dot_exact(k, 2, X1, Y1, s1);
                im = dot_exact(k, 2, X2, Y2, s2);
            } else if (form == 4) {
                /* Eq. 5 with each real GEMM rounded, then the +/- rounded */
                int one = 1;
                xn *P[4]; xn p1, p2, p3, p4;
                p1 = dot_exact(k, 1, (xn *[]){ar}, (xn *[]){br}, &one);
                p2 = dot_exact(k, 1, (xn *[]){ai}, (xn *[]){bi}, &one);
                p3 = dot_exact(k, 1, (xn *[]){ar}, (xn *[]){bi}, &one);
                p4 = dot_exact(k, 1, (xn *[]){ai}, (xn *[]){br}, &one);
                P[0] = &p1; P[1] = &p2; P[2] = &p3; P[3] = &p4;
                xn r[4];
                for (int q = 0; q < 4; q++) r[q] = xn_round(P[q], rounded_prec);
                xn t1 = xn_add(&r[0], &r[1], 1), t2 = xn_add(&r[2], &r[3], 0);
                re = xn_round(&t1, rounded_prec); im = xn_round(&t2, rounded_prec);
                xn_free(&t1); xn_free(&t2);
                for (int q = 0; q < 4; q++) { xn_free(&r[q]); xn_free(P[q]); }
            } else {
                /* Eq. 4 / Eq. 6: T1 = ReA ReB, T2 = ImA ImB, T3 = (ReA+ImA)(ReB+ImB);
                   Re = T1 - T2 ; Im = T3 - T1 - T2 */
                for (int64_t q = 0; q < k; q++) {
                    as[q] = xn_add(&ar[q], &ai[q], 0);
                    bs[q] = xn_add(&br[q], &bi[q], 0);
                    if (rounded_prec) {
                        xn ra = xn_round(&as[q], rounded_prec), rb = xn_round(&bs[q], rounded_prec);
                        xn_free(&as[q]); xn_free(&bs[q]); as[q] = ra; bs[q] = rb;
                    }
                }
                int one = 1;
                xn T1 = dot_exact(k, 1, (xn *[]){ar}, (xn *[]){br}, &one);
                xn T2 = dot_exact(k, 1, (xn *[]){ai}, (xn *[]){bi}, &one);
                xn T3 = dot_exact(k, 1, (xn *[]){as}, (xn *[]){bs}, &one);
                if (rounded_prec) {
                    xn r1 = xn_round(&T1, rounded_prec), r2 = xn_round(&T2, rounded_prec), r3 = xn_round(&T3, rounded_prec);
                    xn_free(&T1); xn_free(&T2); xn_free(&T3); T1 = r1; T2 = r2; T3 = r3;
                }
                xn d = xn_add(&T1, &T2, 1);
                xn u = xn_add(&T3, &T1, 1);
                if (rounded_prec) {
                    re = xn_round(&d, rounded_prec); xn_free(&d);
                    xn ur = xn_round(&u, rounded_prec); xn_free(&u);
                    xn w = xn_add(&ur, &T2, 1); xn_free(&ur);
                    im = xn_round(&w, rounded_prec); xn_free(&w);
                } else {
                    re = d;
                    im = xn_add(&u, &T2, 1); xn_free(&u);
                }
                xn_free(&T1); xn_free(&T2); xn_free(&T3);
                for (int64_t q = 0; q < k; q++) { xn_free(&as[q]); xn_free(&bs[q]); }
            }
            uint8_t *s; int64_t *e; uint64_t *l;
            out_ptrs(Cre, oi, &s, &e, &l); xn_store(&re, prec_out, s, e, l, Cre->L);
            out_ptrs(Cim, oi, &s, &e, &l); xn_store(&im, prec_out, s, e, l, Cim->L);
            xn_free(&re); xn_free(&im);
        }
        free(ar); free(ai); free(br); free(bi); free(as); free(bs);
    }
    return err;
}

/* ------------------------------------------------------------------ oracle (2): Ozaki */
/* mu of Algorithm 2 in exponent form (reading Z3): e = max exponent
 * over the nonzero entries of row i (A, side 0) or column j (B, side 1), common to Re and
 * Im (Z10).  Returns 1 if the row/column has a nonzero entry, else 0 (e=0). */
static int line_exponent(const orc_rmat *Pre, const orc_rmat *Pim, int side, int64_t idx, int64_t len, int64_t *e) {
    int any = 0; int64_t best = 0;
    for (int64_t q = 0; q < len; q++) {
        for (int p = 0; p < 2; p++) {
            const orc_rmat *M = p ? Pim : Pre;
            xn v = side == 0 ? entry_of(M, idx, q) : entry_of(M, q, idx);
            if (!v.n) continue;
            int64_t ex = v.e + 64 * (int64_t)M->L;
            if (!any || ex > best) best = ex;
            any = 1;
        }
    }
    *e = any ? best : 0;
    return any;
}

/* fixed-point value (reading Z5): X = sign * floor(|x| * 2^(W - e)), returned as a two's
 * complement integer in nx limbs.  |x| = N 2^(exp - 64L). */
static void fixed_point(const xn *x, int64_t e, int64_t W, uint64_t *X, int nx) {
    memset(X, 0, sizeof(uint64_t) * (size_t)nx);
    if (!x->n) return;
    int64_t sh = x->e + W - e;        /* X = floor(N * 2^sh) */
    if (sh >= 0) shl_limbs(X, nx, x->m, x->n, sh);
    else shr_limbs(X, nx, x->m, x->n, -sh);
    if (x->neg) {
        uint64_t c = 1;
        for (int i = 0; i < nx; i++) { uint64_t t = ~X[i] + c; c = (c && t == 0); X[i] = t; }
    }
}

static void add_tc(uint64_t *r, const uint64_t *a, const uint64_t *b, int n) {
    uint64_t c = 0;
    for (int i = 0; i < n; i++) { u128 t = (u128)a[i] + b[i] + c; r[i] = (uint64_t)t; c = (uint64_t)(t >> 64); }
}

/* the unique balanced radix-2^b digits (digit set [-2^(b-1), 2^(b-1)-1]) of the two's
 * complement integer X: X = sum_{alpha=1..s} d[alpha-1] 2^(b(s-alpha)).  Slice A_alpha of
 * Algorithm 2 is d[alpha-1] * 2^(e + 3 - b alpha) (b = 8: the INT8 carrier;
 * b = 53 - ceil((53 + ceil(log2 k))/2): the paper's binary64 carrier).  Returns 0 on
 * success, -1 if X does not fit s digits. */
static uint64_t bits_at(const uint64_t *X, int nx, int64_t pos, int b) {   /* b <= 32 */
    int64_t li = pos >> 6; int bo = (int)(pos & 63);
    uint64_t lo = li < nx ? X[li] : (X[nx - 1] >> 63 ? ~0ull : 0ull);
    uint64_t hi = li + 1 < nx ? X[li + 1] : (X[nx - 1] >> 63 ? ~0ull : 0ull);
    uint64_t v = bo ? ((lo >> bo) | (hi << (64 - bo))) : lo;
    return v & ((1ull << b) - 1);
}
static int balanced_digits(const uint64_t *X, int nx, int s, int b, int32_t *d) {
    int64_t c = 0;
    const int64_t half = 1ll << (b - 1), full = 1ll << b;
    for (int t = 0; t < s; t++) {
        int64_t v = (int64_t)bits_at(X, nx, (int64_t)b * t, b) + c;
        int64_t dig = v >= half ? v - full : v;
        c = v >= half;
        d[s - 1 - t] = (int32_t)dig;
    }
    /* the bits above must be the sign extension cancelled by the final carry */
    int neg = (int)(X[nx - 1] >> 63);
    for (int64_t pos = (int64_t)b * s; pos < 64 * (int64_t)nx; pos++) {
        int bit = (int)((X[pos >> 6] >> (pos & 63)) & 1);
        if (bit != neg) return -1;
    }
    return (neg ? (c == 1) : (c == 0)) ? 0 : -1;
}

/* digit planes of one line (row i of A, or column j of B), parts 0 = Re, 1 = Im,
 * 2 = Re + Im (exact fixed-point sum, reading Z11).  dig[part][alpha][q] for q < len. */
static int line_digits(const orc_rmat *Pre, const orc_rmat *Pim, int side, int64_t idx, int64_t len,
                       int64_t e, int s, int b, int nparts, int32_t *dig) {
    int64_t W = (int64_t)b * s - 3;
    int nx = (int)(((int64_t)b * s + 64) / 64 + 1);
    uint64_t X[3][nx];
    int32_t d[s];
    for (int64_t q = 0; q < len; q++) {
        for (int p = 0; p < 2; p++) {
            const orc_rmat *M = p ? Pim : Pre;
            xn v = side == 0 ? entry_of(M, idx, q) : entry_of(M, q, idx);
            fixed_point(&v, e, W, X[p], nx);
        }
        add_tc(X[2], X[0], X[1], nx);
        for (int p = 0; p < nparts; p++) {
            if (balanced_digits(X[p], nx, s, b, d)) return -1;
            for (int a = 0; a < s; a++) dig[((int64_t)p * s + a) * len + q] = d[a];
        }
    }
    return 0;
}

/* Algorithm 2's product for one output element and one (A part, B part):
 * C = sum_{alpha=1..d} sum_{beta=1..d-alpha+1} (A_alpha B_beta)_ij,
 * accumulated exactly (Z7) as the integer  sum (dA_alpha . dB_beta) 2^(b(s+1-alpha-beta))
 * into the two's complement accumulator acc (na limbs, weight 2^(eA+eB+6-b(s+1))). */
static void ozaki_pair(const int32_t *da, const int32_t *db, int64_t k, int s, int b, uint64_t *acc, int na, int neg) {
    /* s here is the triangle's d; the planes da/db may hold more digits (NEXT-4: the top s
       digits of a longer expansion), only alpha, beta <= s are read */
    for (int alpha = 1; alpha <= s; alpha++) {
        const int32_t *xa = da + (int64_t)(alpha - 1) * k;
        for (int beta = 1; beta <= s - alpha + 1; beta++) {
            const int32_t *yb = db + (int64_t)(beta - 1) * k;
            int64_t dot = 0;                                   /* C_alpha,beta := A_alpha B_beta */
            for (int64_t q = 0; q < k; q++) dot += (int64_t)xa[q] * (int64_t)yb[q];
            if (!dot) continue;
            uint64_t mag = (uint64_t)(dot < 0 ? -dot : dot);
            addsh(acc, na, &mag, 1, (int64_t)b * (s + 1 - alpha - beta), neg ^ (dot < 0));
        }
    }
}

/* C := beta * C0 + (alpha_neg ? -1 : +1) * (Ozaki product), every sum exact, ONE RNE (the
 * LU trailing update A22 - L21 U12 of PAPER.md:251, 261 with a single rounding).
 * C0 (Cre0, Cim0) is read at the same positions as the output (full or sampled). */
static int ozaki_core(int64_t m, int64_t n, int64_t k,
                      const orc_rmat *Are, const orc_rmat *Aim, const orc_rmat *Bre, const orc_rmat *Bim,
                      orc_rmat *Cre, orc_rmat *Cim, int32_t prec_out, int32_t form, int32_t s,
                      int64_t nsamp, const int64_t *si, const int64_t *sj, int32_t nthreads,
                      const orc_rmat *Cre0, const orc_rmat *Cim0, int32_t beta, int32_t alpha_neg, int32_t bits,
                      const int32_t *srow);

int orc_cgemm_ozaki(int64_t m, int64_t n, int64_t k,
                    const orc_rmat *Are, const orc_rmat *Aim, const orc_rmat *Bre, const orc_rmat *Bim,
                    orc_rmat *Cre, orc_rmat *Cim, int32_t prec_out, int32_t form, int32_t s,
                    int64_t nsamp, const int64_t *si, const int64_t *sj, int32_t nthreads)
{
    return ozaki_core(m, n, k, Are, Aim, Bre, Bim, Cre, Cim, prec_out, form, s, nsamp, si, sj, nthreads,
                      NULL, NULL, 0, 0, 8, NULL);
}

int orc_cgemm_ozaki_acc(int64_t m, int64_t n, int64_t k,
                        const orc_rmat *Are, const orc_rmat *Aim, const orc_rmat *Bre, const orc_rmat *Bim,
                        const orc_rmat *Cre0, const orc_rmat *Cim0, int32_t beta, int32_t alpha_neg,
                        orc_rmat *Cre, orc_rmat *Cim, int32_t prec_out, int32_t form, int32_t s,
                        int64_t nsamp, const int64_t *si, const int64_t *sj, int32_t nthreads)
{
    return ozaki_core(m, n, k, Are, Aim, Bre, Bim, Cre, Cim, prec_out, form, s, nsamp, si, sj, nthreads,
                      Cre0, Cim0, beta, alpha_neg, 8, NULL);
}

/* the same method with b-bit digits (NEXT-1: b = the paper's binary64 slice width) */
int orc_cgemm_ozaki_bits(int64_t m, int64_t n, int64_t k,
                         const orc_rmat *Are, const orc_rmat *Aim, const orc_rmat *Bre, const orc_rmat *Bim,
                         orc_rmat *Cre, orc_rmat *Cim, int32_t prec_out, int32_t form, int32_t s, int32_t bits,
                         int64_t nsamp, const int64_t *si, const int64_t *sj, int32_t nthreads)
{
    if (bits < 2 || bits > 30) return -1;
    return ozaki_core(m, n, k, Are, Aim, Bre, Bim, Cre, Cim, prec_out, form, s, nsamp, si, sj, nthreads,
                      NULL, NULL, 0, 0, bits, NULL);
}

/* NEXT-4 (the paper's future work "set the optimal number of divisions",
 * PAPER.md:360): a per-row triangle.  Digits are computed once with s_max slices (the split
 * is unchanged); row i uses the TOP srow[i] <= s_max digits of every expansion it touches --
 * its own row's and every column's of B -- and Algorithm 2's triangle with d = srow[i]
 * (PAPER.md:173-177), value P 2^(eA_i + eB_j + 6 - 8(srow[i]+1)), one RNE.  The top t digits
 * of a balanced expansion of X with s_max digits are the balanced digits of
 * floor((X + H) / 256^(s_max-t)), H = sum_{u < s_max-t} 128 256^u (DESIGN.md NEXT-4). */
int orc_cgemm_ozaki_rows(int64_t m, int64_t n, int64_t k,
                         const orc_rmat *Are, const orc_rmat *Aim, const orc_rmat *Bre, const orc_rmat *Bim,
                         orc_rmat *Cre, orc_rmat *Cim, int32_t prec_out, int32_t form, int32_t s_max,
                         const int32_t *srow, int64_t nsamp, const int64_t *si, const int64_t *sj, int32_t nthreads)
{
    if (!srow) return -1;
    for (int64_t i = 0; i < m; i++) if (srow[i] < 1 || srow[i] > s_max) return -1;
    return ozaki_core(m, n, k, Are, Aim, Bre, Bim, Cre, Cim, prec_out, form, s_max, nsamp, si, sj, nthreads,
                      NULL, NULL, 0, 0, 8, srow);
}

/* NEXT-2 + NEXT-4: C := beta C0 +- (per-row-triangle product), one RNE */
int orc_cgemm_ozaki_acc_rows(int64_t m, int64_t n, int64_t k,
                             const orc_rmat *Are, const orc_rmat *Aim, const orc_rmat *Bre, const orc_rmat *Bim,
                             const orc_rmat *Cre0, const orc_rmat *Cim0, int32_t beta, int32_t alpha_neg,
                             orc_rmat *Cre, orc_rmat *Cim, int32_t prec_out, int32_t form, int32_t s_max,
                             const int32_t *srow, int64_t nsamp, const int64_t *si, const int64_t *sj, int32_t nthreads)
{
    if (!srow) return -1;
    for (int64_t i = 0; i < m; i++) if (srow[i] < 1 || srow[i] > s_max) return -1;
    return ozaki_core(m, n, k, Are, Aim, Bre, Bim, Cre, Cim, prec_out, form, s_max, nsamp, si, sj, nthreads,
                      Cre0, Cim0, beta, alpha_neg, 8, srow);
}

/* b = S - ceil((S + ceil(log2 k)) / 2), S = 53: the slice width of Algorithm 2's tau (P:161,
 * reading Z2: ceil(log2 l)); every k-term sum of two b-bit balanced digits is exact in binary64 */
int32_t orc_fp64_slice_bits(int64_t k) {
    int lk = 0; while ((1ll << lk) < k) lk++;
    return 53 - (53 + lk + 1) / 2;
}

static int ozaki_core(int64_t m, int64_t n, int64_t k,
                      const orc_rmat *Are, const orc_rmat *Aim, const orc_rmat *Bre, const orc_rmat *Bim,
                      orc_rmat *Cre, orc_rmat *Cim, int32_t prec_out, int32_t form, int32_t s,
                      int64_t nsamp, const int64_t *si, const int64_t *sj, int32_t nthreads,
                      const orc_rmat *Cre0, const orc_rmat *Cim0, int32_t beta, int32_t alpha_neg, int32_t bits,
                      const int32_t *srow)
{
    if (m < 0 || n < 0 || k < 0 || (form != 3 && form != 4) || s < 1 || prec_out < 2) return -1;
    int64_t total = nsamp < 0 ? m * n : nsamp;
    int nt = nthreads_of(nthreads);
    int nparts = form == 3 ? 3 : 2;
    int err = 0;
    int cnt = 2; while ((1LL << cnt) < 4 * k + 1) cnt++;
    const int b = bits;
    int na = (int)(((int64_t)b * s + 2 * b + cnt + 64) / 64 + 2);
    #pragma omp parallel num_threads(nt)
    {
        int32_t *da = (int32_t *)malloc(sizeof(int32_t) * (size_t)nparts * s * (k ? k : 1));
        int32_t *db = (int32_t *)malloc(sizeof(int32_t) * (size_t)nparts * s * (k ? k : 1));
        uint64_t *acc[3];
        for (int q = 0; q < 3; q++) acc[q] = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)na);
        #pragma omp for schedule(dynamic, 1)
        for (int64_t t = 0; t < total; t++) {
            int64_t i = nsamp < 0 ? t / (n ? n : 1) : si[t];
            int64_t j = nsamp < 0 ? t % (n ? n : 1) : sj[t];
            int64_t oi = nsamp < 0 ? i * Cre->ld + j : t;
            if (i < 0 || i >= m || j < 0 || j >= n) { err = -1; continue; }
            int64_t eA, eB;
            line_exponent(Are, Aim, 0, i, k, &eA);
            line_exponent(Bre, Bim, 1, j, k, &eB);
            if (line_digits(Are, Aim, 0, i, k, eA, s, b, nparts, da) ||
                line_digits(Bre, Bim, 1, j, k, eB, s, b, nparts, db)) { err = -2; continue; }
            const int64_t pl = (int64_t)s * k;
            const int d = srow ? srow[i] : s;             /* the triangle's d for this row */
            for (int q = 0; q < 3; q++) memset(acc[q], 0, sizeof(uint64_t) * (size_t)na);
            if (form == 4) {
                /* Eq. 5: Re = ReA ReB - ImA ImB ; Im = ReA ImB + ImA ReB  (each by Alg. 2) */
                ozaki_pair(da, db, k, d, b, acc[0], na, 0);
                ozaki_pair(da + pl, db + pl, k, d, b, acc[0], na, 1);
                ozaki_pair(da, db + pl, k, d, b, acc[1], na, 0);
                ozaki_pair(da + pl, db, k, d, b, acc[1], na, 0);
            } else {
                /* Eq. 6: T1 = ReA ReB, T2 = ImA ImB, T3 = (ReA+ImA)(ReB+ImB) (each by Alg. 2);
                   Re = T1 - T2 ; Im = T3 - T1 - T2 */
                ozaki_pair(da, db, k, d, b, acc[0], na, 0);                /* T1 */
                ozaki_pair(da + pl, db + pl, k, d, b, acc[1], na, 0);      /* T2 */
                ozaki_pair(da + 2 * pl, db + 2 * pl, k, d, b, acc[2], na, 0); /* T3 */
            }
            int64_t e0 = eA + eB + 6 - (int64_t)b * (d + 1);
            xn re, im;
            if (form == 4) {
                re = xn_from_acc(acc[0], na, e0);
                im = xn_from_acc(acc[1], na, e0);
            } else {
                xn T1 = xn_from_acc(acc[0], na, e0), T2 = xn_from_acc(acc[1], na, e0), T3 = xn_from_acc(acc[2], na, e0);
                re = xn_add(&T1, &T2, 1);
                xn u = xn_add(&T3, &T1, 1);
                im = xn_add(&u, &T2, 1);
                xn_free(&u); xn_free(&T1); xn_free(&T2); xn_free(&T3);
            }
            if (alpha_neg) { re.neg = re.n ? !re.neg : 0; im.neg = im.n ? !im.neg : 0; }
            if (beta) {                                   /* exact C0 + (+-P), then one rounding */
                xn c0r = entry_of(Cre0, i, j), c0i = entry_of(Cim0, i, j);
                xn sr = xn_add(&c0r, &re, 0), sm = xn_add(&c0i, &im, 0);
                xn_free(&re); xn_free(&im);
                re = sr; im = sm;
            }
            uint8_t *sg; int64_t *ex; uint64_t *lb;
            out_ptrs(Cre, oi, &sg, &ex, &lb); xn_store(&re, prec_out, sg, ex, lb, Cre->L);
            out_ptrs(Cim, oi, &sg, &ex, &lb); xn_store(&im, prec_out, sg, ex, lb, Cim->L);
            xn_free(&re); xn_free(&im);
        }
        free(da); free(db);
        for (int q = 0; q < 3; q++) free(acc[q]);
    }
    return err;
}

/* exponents eA[m] (rows of A), eB[n] (columns of B) and nonzero flags */
int orc_exponents(int64_t m, int64_t n, int64_t k,
                  const orc_rmat *Are, const orc_rmat *Aim, const orc_rmat *Bre, const orc_rmat *Bim,
                  int64_t *eA, int64_t *eB, uint8_t *nzA, uint8_t *nzB)
{
    for (int64_t i = 0; i < m; i++) nzA[i] = (uint8_t)line_exponent(Are, Aim, 0, i, k, &eA[i]);
    for (int64_t j = 0; j < n; j++) nzB[j] = (uint8_t)line_exponent(Bre, Bim, 1, j, k, &eB[j]);
    return 0;
}

/* digit planes (slices of Algorithm 2 under the readings) of A (side 0: dig[part][alpha][i][q],
 * q < k) or B (side 1: dig[part][alpha][j][q], i.e. column j of B as a line).  nparts = 2
 * (Re, Im) or 3 (Re, Im, Re+Im). */
int orc_split_bits(int side, int64_t rows, int64_t k, const orc_rmat *Pre, const orc_rmat *Pim,
                   int32_t s, int32_t bits, int32_t nparts, int32_t *dig)
{
    int32_t *tmp = (int32_t *)malloc(sizeof(int32_t) * (size_t)nparts * s * (k ? k : 1));
    int rc = 0;
    for (int64_t r = 0; r < rows && !rc; r++) {
        int64_t e;
        line_exponent(Pre, Pim, side, r, k, &e);
        if (line_digits(Pre, Pim, side, r, k, e, s, bits, nparts, tmp)) { rc = -2; break; }
        for (int p = 0; p < nparts; p++)
            for (int a = 0; a < s; a++)
                memcpy(dig + (((int64_t)p * s + a) * rows + r) * k, tmp + ((int64_t)p * s + a) * k, sizeof(int32_t) * (size_t)k);
    }
    free(tmp);
    return rc;
}

int orc_split(int side, int64_t rows, int64_t k, const orc_rmat *Pre, const orc_rmat *Pim,
              int32_t s, int32_t nparts, int8_t *dig)
{
    int32_t *d32 = (int32_t *)malloc(sizeof(int32_t) * (size_t)nparts * s * (rows ? rows : 1) * (k ? k : 1));
    int rc = orc_split_bits(side, rows, k, Pre, Pim, s, 8, nparts, d32);
    for (int64_t q = 0; q < (int64_t)nparts * s * rows * k; q++) dig[q] = (int8_t)d32[q];
    free(d32);
    return rc;
}

/* ------------------------------------------------------------------ slice-count rule */
/* t = floor(max(|Re|,|Im|) * 2^(7 - e)) in [0,127] for one entry */
static int top7(const orc_rmat *Pre, const orc_rmat *Pim, int side, int64_t idx, int64_t q, int64_t e) {
    int best = 0;
    for (int p = 0; p < 2; p++) {
        const orc_rmat *M = p ? Pim : Pre;
        xn v = side == 0 ? entry_of(M, idx, q) : entry_of(M, q, idx);
        if (!v.n) continue;
        uint64_t X[2];
        int64_t sh = v.e + 7 - e;
        if (sh >= 0) shl_limbs(X, 2, v.m, v.n, sh); else shr_limbs(X, 2, v.m, v.n, -sh);
        int t = (int)X[0];
        if (X[1] || X[0] > 127) return -1;    /* cannot happen for exp <= e */
        if (t > best) best = t;
    }
    return best;
}

/* entry exponent for the max-plus bound: max(exp Re, exp Im) over the nonzero parts,
 * so |a| >= 2^(e-1); returns 0 if the entry is zero */
static int entry_mpexp(const orc_rmat *Pre, const orc_rmat *Pim, int side, int64_t idx, int64_t q, int64_t *e) {
    int any = 0;
    for (int p = 0; p < 2; p++) {
        const orc_rmat *M = p ? Pim : Pre;
        xn v = side == 0 ? entry_of(M, idx, q) : entry_of(M, q, idx);
        if (!v.n) continue;
        int64_t ex = v.e + 64 * (int64_t)M->L;
        if (!any || ex > *e) *e = ex;
        any = 1;
    }
    return any;
}

/* The rho-hat pre-pass.  Over the pairs (i, j) of a nonzero row
 * of A and a nonzero column of B:
 *   T_ij  = sum_k t_ik u_kj   (bound 1: rho_ij <= k 2^14 / T_ij when T_ij > 0)
 *   D_ij  = eA_i + eB_j - max_k (e_ik + e_kj)   over k with a_ik, b_kj both nonzero
 *           (bound 2: rho_ij <= k 2^(2 + D_ij); no such k <=> (|A||B|)_ij = 0, pair skipped)
 * out[0] = min_ij T_ij (-1: no pair).  If out[0] == 0 the combined rule needs, with each
 * pair assigned to bound 2 iff T_ij == 0 or (D_ij < 12 and T_ij 2^D_ij < 2^12):
 * out[1] = min T_ij over bound-1 pairs (-1: none), out[2] = max D_ij over bound-2 pairs
 * (-1: none).  When out[0] != 0 and !full, out[1] = out[0] and out[2] = -1 (full: the
 * bound-1 / bound-2 split is always reported; used by multi-rank reductions). */
int orc_rho_bounds(int64_t m, int64_t n, int64_t k,
                   const orc_rmat *Are, const orc_rmat *Aim, const orc_rmat *Bre, const orc_rmat *Bim,
                   int64_t *out, int32_t nthreads, int32_t full)
{
    int64_t *eA = (int64_t *)malloc(sizeof(int64_t) * (size_t)(m + 1)), *eB = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
    uint8_t *nzA = (uint8_t *)malloc((size_t)m + 1), *nzB = (uint8_t *)malloc((size_t)n + 1);
    int32_t *t = (int32_t *)malloc(sizeof(int32_t) * (size_t)(m * k + 1));
    int32_t *u = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n * k + 1));
    int64_t *ea = (int64_t *)malloc(sizeof(int64_t) * (size_t)(m * k + 1));
    int64_t *eb = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n * k + 1));
    uint8_t *za = (uint8_t *)malloc((size_t)(m * k + 1)), *zb = (uint8_t *)malloc((size_t)(n * k + 1));
    orc_exponents(m, n, k, Are, Aim, Bre, Bim, eA, eB, nzA, nzB);
    int rc = 0;
    for (int64_t i = 0; i < m; i++) for (int64_t q = 0; q < k; q++) {
        int v = top7(Are, Aim, 0, i, q, eA[i]); if (v < 0) rc = -2; t[i * k + q] = v;
        za[i * k + q] = (uint8_t)entry_mpexp(Are, Aim, 0, i, q, &ea[i * k + q]); }
    for (int64_t j = 0; j < n; j++) for (int64_t q = 0; q < k; q++) {
        int v = top7(Bre, Bim, 1, j, q, eB[j]); if (v < 0) rc = -2; u[j * k + q] = v;
        zb[j * k + q] = (uint8_t)entry_mpexp(Bre, Bim, 1, j, q, &eb[j * k + q]); }
    int nt = nthreads_of(nthreads);
    int64_t mn = -1, mn1 = -1, mx2 = -1;
    #pragma omp parallel num_threads(nt)
    {
        int64_t loc = -1, loc1 = -1, loc2 = -1;
        #pragma omp for schedule(dynamic, 1)
        for (int64_t i = 0; i < m; i++) {
            if (!nzA[i]) continue;
            for (int64_t j = 0; j < n; j++) {
                if (!nzB[j]) continue;
                int64_t T = 0, mp = 0; int has = 0;
                for (int64_t q = 0; q < k; q++) {
                    T += (int64_t)t[i * k + q] * u[j * k + q];
                    if (za[i * k + q] && zb[j * k + q]) {
                        int64_t x = ea[i * k + q] + eb[j * k + q];
                        if (!has || x > mp) mp = x;
                        has = 1;
                    }
                }
                if (!has) continue;                     /* (|A||B|)_ij = 0: C_ij = 0 exactly */
                if (loc < 0 || T < loc) loc = T;
                int64_t D = eA[i] + eB[j] - mp;
                int use2 = (T == 0) || (D < 12 && (T << D) < 4096);
                if (use2) { if (D > loc2) loc2 = D; }
                else if (loc1 < 0 || T < loc1) loc1 = T;
            }
        }
        #pragma omp critical
        {
            if (loc >= 0 && (mn < 0 || loc < mn)) mn = loc;
            if (loc1 >= 0 && (mn1 < 0 || loc1 < mn1)) mn1 = loc1;
            if (loc2 > mx2) mx2 = loc2;
        }
    }
    out[0] = mn;
    if (mn != 0 && !full) { out[1] = mn; out[2] = -1; } else { out[1] = mn1; out[2] = mx2; }
    free(eA); free(eB); free(nzA); free(nzB); free(t); free(u); free(ea); free(eb); free(za); free(zb);
    return rc;
}

/* the slice-count rule from the pre-pass integers:
 *   minT > 0 : log2rho = log2((double)k) + 14.0 - log2((double)minT)
 *   minT == 0: log2rho = max( log2((double)k) + 14.0 - log2((double)minT1)   [minT1 >= 1],
 *                             log2((double)k) + 2.0 + (double)maxD2 )          [maxD2 >= 0]
 *   minT < 0 : log2rho = 0 (the product is identically zero)
 *   s = min{ s >= 1 : 8.0 s >= prec - 4.0 + log2(c_M s) + log2rho + 0.1 }, c_4M = 3, c_3M = 4 */
int32_t orc_slices_for_bits(int32_t prec, int32_t form, int64_t k, int64_t minT, int64_t minT1, int64_t maxD2,
                            int32_t bits);
int32_t orc_slices_for(int32_t prec, int32_t form, int64_t k, int64_t minT, int64_t minT1, int64_t maxD2) {
    return orc_slices_for_bits(prec, form, k, minT, minT1, maxD2, 8);
}
/* the rule with b-bit digits: min{ s : b s >= prec - 4 + log2(c_M s) + log2rho + 0.1 } */
int32_t orc_slices_for_bits(int32_t prec, int32_t form, int64_t k, int64_t minT, int64_t minT1, int64_t maxD2,
                            int32_t bits) {
    double c = form == 3 ? 4.0 : 3.0;
    double log2rho = 0.0;
    if (minT > 0) log2rho = log2((double)k) + 14.0 - log2((double)minT);
    else if (minT == 0) {
        log2rho = -1e300;
        if (minT1 >= 1) log2rho = log2((double)k) + 14.0 - log2((double)minT1);
        if (maxD2 >= 0) { double b2 = log2((double)k) + 2.0 + (double)maxD2; if (b2 > log2rho) log2rho = b2; }
        if (log2rho < -1e299) log2rho = 0.0;
    }
    for (int32_t s = 1; s < 1000000; s++)
        if ((double)bits * s >= (double)prec - 4.0 + log2(c * s) + log2rho + 0.1) return s;
    return -1;
}

/* ================================================================== NEXT-3: complex LU
 * The paper's second workload (Eq. 7, Fig. 3): blocked right-looking complex
 * LU with partial pivoting whose trailing update A22 := A22 - L21 U12 is an Ozaki complex GEMM
 * ("For fast LU decomposition, L21 U12 must be fast in xGEMM"), plus the forward
 * and backward substitutions of Eq. 7.  Scalar operations are MPC-style: each real part of a
 * complex result is the exact value rounded ONCE to prec (RNE; reading Z8):
 *   cmul(x, y)    = ( RNE(xr yr - xi yi), RNE(xr yi + xi yr) )
 *   cfms(a, x, y) = ( RNE(ar - (xr yr - xi yi)), RNE(ai - (xr yi + xi yr)) )      a - x y
 *   crecip(z)     = ( RNE(zr / (zr^2 + zi^2)), RNE(-zi / (zr^2 + zi^2)) )
 * The column scaling multiplies by the rounded reciprocal of the pivot (as LAPACK's xGETF2
 * scales by 1 / A(j,j)), and the back substitution x_c = cmul(y_c, crecip(u_cc)).
 * Pivot (max |re| + |im|): key(z) = (e, v), e = max exponent of the nonzero
 * parts, v = t(re) + t(im) in binary64 (round to nearest), t(x) = (top 53 bits of |x|,
 * truncated) * 2^(exp(x) - e) as a binary64 (0 if exp(x) - e < -1000); keys compare by (e, v)
 * after normalising v into [0.5, 1) (v >= 1: e + 1, v / 2).  First maximum wins. */

static xn xn_mul(const xn *a, const xn *b) {
    xn r = {0, 0, 0, NULL, 1};
    if (!a->n || !b->n) { r.own = 0; return r; }
    r.m = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(a->n + b->n));
    mulmag(r.m, a->m, a->n, b->m, b->n);
    r.n = a->n + b->n;
    r.e = a->e + b->e;
    r.neg = a->neg ^ b->neg;
    return r;
}

/* RNE(a / b) to prec bits (b != 0): q = floor(Na 2^sh / Nb) with >= prec + 2 bits by plain
 * shift-and-subtract long division, then RNE of 2 q + (remainder != 0) */
static void xn_div_store(const xn *a, const xn *b, int prec, uint8_t *sign, int64_t *exp, uint64_t *limbs, int Lout) {
    if (!a->n) { xn z = {0, 0, 0, NULL, 0}; xn_store(&z, prec, sign, exp, limbs, Lout); return; }
    int ba = bitlen_limbs(a->m, a->n), bb = bitlen_limbs(b->m, b->n);
    int64_t sh = (int64_t)prec + 2 + bb - ba;            /* Na 2^sh >= 2^(prec+1) Nb */
    if (sh < 0) sh = 0;
    int nn = (int)((ba + sh) / 64) + 2, nd = b->n + 1;
    uint64_t *num = (uint64_t *)calloc((size_t)nn, 8), *q = (uint64_t *)calloc((size_t)nn + 1, 8);
    uint64_t *rem = (uint64_t *)calloc((size_t)nd + 1, 8);
    shl_limbs(num, nn, a->m, a->n, sh);
    for (int64_t pos = 64 * (int64_t)nn - 1; pos >= 0; pos--) {
        uint64_t c = (uint64_t)getbit(num, nn, pos);        /* rem = 2 rem + bit */
        for (int i = 0; i <= nd; i++) { uint64_t t = rem[i] >> 63; rem[i] = (rem[i] << 1) | c; c = t; }
        int ge = 1;                                          /* rem >= Nb ? */
        for (int i = nd; i >= 0; i--) {
            uint64_t d = i < b->n ? b->m[i] : 0;
            if (rem[i] != d) { ge = rem[i] > d; break; }
        }
        if (ge) {
            uint64_t br = 0;
            for (int i = 0; i <= nd; i++) {
                uint64_t d = i < b->n ? b->m[i] : 0;
                u128 t = (u128)rem[i] - d - br;
                rem[i] = (uint64_t)t; br = (t >> 64) ? 1 : 0;
            }
            q[pos >> 6] |= 1ull << (pos & 63);
        }
    }
    int sticky = !is_zero_limbs(rem, nd + 1);
    xn r; r.own = 1; r.n = nn + 1; r.m = (uint64_t *)calloc((size_t)nn + 1, 8);
    shl_limbs(r.m, nn + 1, q, nn, 1);
    r.m[0] |= (uint64_t)sticky;
    r.e = a->e - b->e - sh - 1;
    r.neg = a->neg ^ b->neg;
    xn_store(&r, prec, sign, exp, limbs, Lout);
    xn_free(&r); free(num); free(q); free(rem);
}

static xn xn_of(const uint8_t *s, const int64_t *e, const uint64_t *l, int L) {
    xn v; v.m = (uint64_t *)l; v.n = is_zero_limbs(l, L) ? 0 : L; v.neg = v.n ? (*s != 0) : 0;
    v.e = *e - 64 * (int64_t)L; v.own = 0;
    return v;
}

typedef struct { uint8_t *s; int64_t *e; uint64_t *l; } orc_el;     /* one real element */
static orc_el el_at(orc_rmat *M, int64_t r, int64_t c) {
    int64_t idx = r * M->ld + c;
    orc_el x = {M->sign + idx, M->exp + idx, M->limbs + idx * M->L};
    return x;
}
static xn xn_el(orc_el x, int L) { return xn_of(x.s, x.e, x.l, L); }

/* (or, oi) := a - x y  (a may be NULL: := x y) , each part one RNE */
static void c_fms(int L, int prec, const xn *ar, const xn *ai, const xn *xr, const xn *xi,
                  const xn *yr, const xn *yi, orc_el or_, orc_el oi) {
    xn p1 = xn_mul(xr, yr), p2 = xn_mul(xi, yi), p3 = xn_mul(xr, yi), p4 = xn_mul(xi, yr);
    xn re = xn_add(&p1, &p2, 1), im = xn_add(&p3, &p4, 0);
    if (ar) {
        xn r2 = xn_add(ar, &re, 1), i2 = xn_add(ai, &im, 1);
        xn_free(&re); xn_free(&im); re = r2; im = i2;
    }
    xn_store(&re, prec, or_.s, or_.e, or_.l, L);
    xn_store(&im, prec, oi.s, oi.e, oi.l, L);
    xn_free(&p1); xn_free(&p2); xn_free(&p3); xn_free(&p4); xn_free(&re); xn_free(&im);
}

static void c_recip(int L, int prec, const xn *zr, const xn *zi, orc_el or_, orc_el oi) {
    xn a = xn_mul(zr, zr), b = xn_mul(zi, zi);
    xn d = xn_add(&a, &b, 0);
    xn nzi = *zi; nzi.neg = nzi.n ? !nzi.neg : 0;
    xn_div_store(zr, &d, prec, or_.s, or_.e, or_.l, L);
    xn_div_store(&nzi, &d, prec, oi.s, oi.e, oi.l, L);
    xn_free(&a); xn_free(&b); xn_free(&d);
}

/* top 53 bits of |x| (truncated) as a binary64 scaled by 2^(exp - e) */
static double key_part(const xn *x, int64_t e) {
    if (!x->n) return 0.0;
    int b = bitlen_limbs(x->m, x->n);
    int64_t ex = x->e + b;                       /* MPFR exponent */
    if (ex - e < -1000) return 0.0;
    uint64_t t;
    shr_limbs(&t, 1, x->m, x->n, b - 53);
    return ldexp((double)t, (int)(ex - e - 53));
}
static void pivot_key(const xn *re, const xn *im, int64_t *e, double *v) {
    int any = 0; int64_t best = 0;
    const xn *p[2] = {re, im};
    for (int q = 0; q < 2; q++) {
        if (!p[q]->n) continue;
        int64_t ex = p[q]->e + bitlen_limbs(p[q]->m, p[q]->n);
        if (!any || ex > best) best = ex;
        any = 1;
    }
    if (!any) { *e = INT64_MIN; *v = 0.0; return; }
    volatile double a = key_part(re, best), b = key_part(im, best);
    double s = a + b;
    if (s >= 1.0) { s = s * 0.5; best += 1; }
    *e = best; *v = s;
}

/* elementwise scalar ops for the pins: op 0 = cmul(x, y), 1 = cfms(a, x, y), 2 = crecip(x),
 * 3 = pivot key (written to kv[2*i] = e, kv[2*i+1] = v bits).  All matrices 1 x cnt. */
int orc_cscalar(int32_t op, int64_t cnt, int32_t prec, const orc_rmat *Ar, const orc_rmat *Ai,
                const orc_rmat *Xr, const orc_rmat *Xi, const orc_rmat *Yr, const orc_rmat *Yi,
                orc_rmat *Or, orc_rmat *Oi, int64_t *kv)
{
    int L = Xr->L;
    for (int64_t t = 0; t < cnt; t++) {
        xn xr = entry_of(Xr, 0, t), xi = entry_of(Xi, 0, t);
        if (op == 3) {
            double v; pivot_key(&xr, &xi, &kv[2 * t], &v);
            memcpy(&kv[2 * t + 1], &v, 8);
            continue;
        }
        orc_el o1 = el_at(Or, 0, t), o2 = el_at(Oi, 0, t);
        if (op == 2) { if (!xr.n && !xi.n) return -1; c_recip(L, prec, &xr, &xi, o1, o2); continue; }
        xn yr = entry_of(Yr, 0, t), yi = entry_of(Yi, 0, t);
        if (op == 0) c_fms(L, prec, NULL, NULL, &xr, &xi, &yr, &yi, o1, o2);
        else { xn ar = entry_of(Ar, 0, t), ai = entry_of(Ai, 0, t); c_fms(L, prec, &ar, &ai, &xr, &xi, &yr, &yi, o1, o2); }
    }
    return 0;
}

static orc_rmat view(const orc_rmat *M, int64_t r, int64_t c) {
    orc_rmat v = *M;
    int64_t idx = r * M->ld + c;
    v.sign = M->sign + idx; v.exp = M->exp + idx; v.limbs = M->limbs + idx * M->L;
    return v;
}

static void swap_rows(orc_rmat *M, int64_t r1, int64_t r2, int64_t ncols) {
    int L = M->L;
    for (int64_t c = 0; c < ncols; c++) {
        orc_el a = el_at(M, r1, c), b = el_at(M, r2, c);
        uint8_t ts = *a.s; *a.s = *b.s; *b.s = ts;
        int64_t te = *a.e; *a.e = *b.e; *b.e = te;
        for (int l = 0; l < L; l++) { uint64_t x = a.l[l]; a.l[l] = b.l[l]; b.l[l] = x; }
    }
}

/* In place: L (unit lower, strictly below the diagonal) and U (upper) with P A = L U;
 * ipiv[c] = the row swapped with row c at step c.  For each panel j0 = 0, K, 2K, ... of width
 * w = min(K, n - j0) (Fig. 3):
 *   (a) for c in [j0, j0+w): pivot p = argmax_{r >= c} key(A_rc); swap rows c, p (all
 *       columns); r = crecip(A_cc); A_rc := cmul(A_rc, r) for r > c; A_rt := cfms(A_rt, A_rc,
 *       A_ct) for r > c, c < t < j0+w                               (panel, LAPACK xGETF2)
 *   (b) for c in [j0, j0+w), r in (c, j0+w), t >= j0+w: A_rt := cfms(A_rt, A_rc, A_ct)
 *                                                                    (U12 := L11^-1 A12)
 *   (c) A22 := A22 - L21 U12 by orc_cgemm_ozaki_acc (form, certified s of this product, one
 *       rounding per element)
 * Returns 0, or c + 1 for the first zero pivot (the factorization continues), < 0 on error.
 * smax (optional) receives the largest slice count used by the updates. */
int orc_clu_factor(int64_t n, orc_rmat *Ar, orc_rmat *Ai, int32_t prec, int32_t K, int32_t form,
                   int64_t *ipiv, int32_t nthreads, int32_t *smax)
{
    if (n < 0 || K < 1 || (form != 3 && form != 4)) return -1;
    const int L = Ar->L;
    int info = 0;
    if (smax) *smax = 0;
    for (int64_t j0 = 0; j0 < n; j0 += K) {
        const int64_t w = (n - j0 < K) ? n - j0 : K;
        for (int64_t c = j0; c < j0 + w; c++) {
            int64_t p = c, be = INT64_MIN; double bv = 0.0;
            for (int64_t r = c; r < n; r++) {
                xn zr = xn_el(el_at(Ar, r, c), L), zi = xn_el(el_at(Ai, r, c), L);
                int64_t e; double v;
                pivot_key(&zr, &zi, &e, &v);
                if (e > be || (e == be && v > bv)) { be = e; bv = v; p = r; }
            }
            ipiv[c] = p;
            if (p != c) { swap_rows(Ar, c, p, n); swap_rows(Ai, c, p, n); }
            xn pr = xn_el(el_at(Ar, c, c), L), pi = xn_el(el_at(Ai, c, c), L);
            if (!pr.n && !pi.n) { if (!info) info = (int)(c + 1); continue; }
            uint8_t rs[2]; int64_t re_[2]; uint64_t rl[2][64];
            orc_el o1 = {&rs[0], &re_[0], rl[0]}, o2 = {&rs[1], &re_[1], rl[1]};
            c_recip(L, prec, &pr, &pi, o1, o2);
            xn rr = xn_el(o1, L), ri = xn_el(o2, L);
            for (int64_t r = c + 1; r < n; r++) {
                xn ar = xn_el(el_at(Ar, r, c), L), ai = xn_el(el_at(Ai, r, c), L);
                c_fms(L, prec, NULL, NULL, &ar, &ai, &rr, &ri, el_at(Ar, r, c), el_at(Ai, r, c));
            }
            #pragma omp parallel for num_threads(nthreads_of(nthreads)) schedule(static)
            for (int64_t r = c + 1; r < n; r++) {
                xn lr = xn_el(el_at(Ar, r, c), L), li = xn_el(el_at(Ai, r, c), L);
                for (int64_t t = c + 1; t < j0 + w; t++) {
                    xn ur = xn_el(el_at(Ar, c, t), L), ui = xn_el(el_at(Ai, c, t), L);
                    xn ar = xn_el(el_at(Ar, r, t), L), ai = xn_el(el_at(Ai, r, t), L);
                    c_fms(L, prec, &ar, &ai, &lr, &li, &ur, &ui, el_at(Ar, r, t), el_at(Ai, r, t));
                }
            }
        }
        if (j0 + w >= n) break;
        for (int64_t c = j0; c < j0 + w; c++) {
            #pragma omp parallel for num_threads(nthreads_of(nthreads)) schedule(static)
            for (int64_t t = j0 + w; t < n; t++) {
                xn ur = xn_el(el_at(Ar, c, t), L), ui = xn_el(el_at(Ai, c, t), L);
                for (int64_t r = c + 1; r < j0 + w; r++) {
                    xn lr = xn_el(el_at(Ar, r, c), L), li = xn_el(el_at(Ai, r, c), L);
                    xn ar = xn_el(el_at(Ar, r, t), L), ai = xn_el(el_at(Ai, r, t), L);
                    c_fms(L, prec, &ar, &ai, &lr, &li, &ur, &ui, el_at(Ar, r, t), el_at(Ai, r, t));
                }
            }
        }
        const int64_t m2 = n - j0 - w;
        orc_rmat L21r = view(Ar, j0 + w, j0), L21i = view(Ai, j0 + w, j0);
        orc_rmat U12r = view(Ar, j0, j0 + w), U12i = view(Ai, j0, j0 + w);
        orc_rmat A22r = view(Ar, j0 + w, j0 + w), A22i = view(Ai, j0 + w, j0 + w);
        int64_t rb[3];
        if (orc_rho_bounds(m2, m2, w, &L21r, &L21i, &U12r, &U12i, rb, nthreads, 0)) return -2;
        int32_t s = orc_slices_for(prec, form, w, rb[0], rb[1], rb[2]);
        if (s < 1) return -3;
        if (smax && s > *smax) *smax = s;
        if (ozaki_core(m2, m2, w, &L21r, &L21i, &U12r, &U12i, &A22r, &A22i, prec, form, s, -1, NULL, NULL,
                       nthreads, &A22r, &A22i, 1, 1, 8, NULL))
            return -4;
    }
    return info;
}

/* Eq. 7 with the factors of orc_clu_factor: B (n x nrhs) := A^-1 B.  Row swaps ipiv[c] in
 * order; forward substitution B_r := cfms(B_r, L_rc, B_c) (r > c, c ascending); backward
 * B_c := cmul(B_c, crecip(U_cc)), then B_r := cfms(B_r, U_rc, B_c) (r < c, c descending). */
int orc_clu_solve(int64_t n, const orc_rmat *LUr, const orc_rmat *LUi, const int64_t *ipiv,
                  orc_rmat *Br, orc_rmat *Bi, int64_t nrhs, int32_t prec)
{
    const int L = LUr->L;
    orc_rmat *Mr = (orc_rmat *)LUr, *Mi = (orc_rmat *)LUi;
    for (int64_t c = 0; c < n; c++)
        if (ipiv[c] != c) { swap_rows(Br, c, ipiv[c], nrhs); swap_rows(Bi, c, ipiv[c], nrhs); }
    for (int64_t c = 0; c < n; c++)
        for (int64_t r = c + 1; r < n; r++) {
            xn lr = xn_el(el_at(Mr, r, c), L), li = xn_el(el_at(Mi, r, c), L);
            for (int64_t q = 0; q < nrhs; q++) {
                xn yr = xn_el(el_at(Br, c, q), L), yi = xn_el(el_at(Bi, c, q), L);
                xn ar = xn_el(el_at(Br, r, q), L), ai = xn_el(el_at(Bi, r, q), L);
                c_fms(L, prec, &ar, &ai, &lr, &li, &yr, &yi, el_at(Br, r, q), el_at(Bi, r, q));
            }
        }
    for (int64_t c = n - 1; c >= 0; c--) {
        xn ur = xn_el(el_at(Mr, c, c), L), ui = xn_el(el_at(Mi, c, c), L);
        if (!ur.n && !ui.n) return -1;
        uint8_t rs[2]; int64_t re_[2]; uint64_t rl[2][64];
        orc_el o1 = {&rs[0], &re_[0], rl[0]}, o2 = {&rs[1], &re_[1], rl[1]};
        c_recip(L, prec, &ur, &ui, o1, o2);
        xn rr = xn_el(o1, L), ri = xn_el(o2, L);
        for (int64_t q = 0; q < nrhs; q++) {
            xn yr = xn_el(el_at(Br, c, q), L), yi = xn_el(el_at(Bi, c, q), L);
            c_fms(L, prec, NULL, NULL, &yr, &yi, &rr, &ri, el_at(Br, c, q), el_at(Bi, c, q));
        }
        for (int64_t r = 0; r < c; r++) {
            xn lr = xn_el(el_at(Mr, r, c), L), li = xn_el(el_at(Mi, r, c), L);
            for (int64_t q = 0; q < nrhs; q++) {
                xn yr = xn_el(el_at(Br, c, q), L), yi = xn_el(el_at(Bi, c, q), L);
                xn ar = xn_el(el_at(Br, r, q), L), ai = xn_el(el_at(Bi, r, q), L);
                c_fms(L, prec, &ar, &ai, &lr, &li, &yr, &yi, el_at(Br, r, q), el_at(Bi, r, q));
            }
        }
    }
    return 0;
}
