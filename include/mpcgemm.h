/* mpcgemm.h -- C ABI of the B200 (sm_100a) Ozaki-scheme complex multiple-precision GEMM.
 *
 * Operation (Eq. 1):  C := A B,  A in C^{m x k}, B in C^{k x n}, with the
 * complex product formed by the 4M method (Eq. 5) or the 3M method
 * (Eq. 6), and every real product computed by the Ozaki scheme
 * (Algorithm 2) on INT8 tensor cores.  DESIGN.md states the readings
 * (Z1..Z24) under which the result is defined; it is bit-identical to oracle/mpref.c
 * orc_cgemm_ozaki() for the same s:
 *
 *   eA_i = max exponent over the nonzero entries of row i of Re A and Im A    (mu_A)
 *   eB_j = max exponent over the nonzero entries of column j of Re B, Im B   (mu_B)
 *   W = 8 s - 3;  X(x) = sign(x) floor(|x| 2^(W - e))  (e = eA_i or eB_j)
 *   slices: X = sum_{alpha=1..s} d_alpha 256^(s-alpha), d_alpha in [-128,127] (unique
 *           balanced radix-256 digits); 3M sums use X(Re) + X(Im) exactly
 *   real product P = sum_{alpha+beta <= s+1} (D^A_alpha D^B_beta) 256^(s+1-alpha-beta)
 *           exact in integers, value P * 2^(eA_i + eB_j + 6 - 8(s+1))
 *   4M: Re = P(ReA,ReB) - P(ImA,ImB), Im = P(ReA,ImB) + P(ImA,ReB)
 *   3M: T1 = P(ReA,ReB), T2 = P(ImA,ImB), T3 = P(ReA+ImA, ReB+ImB), Re = T1 - T2, Im = T3 - T1 - T2
 *   output: each part rounded once to nearest-even at prec bits.
 *
 * Element format (MPFR convention; planar complex):
 *   value = (-1)^sign * N * 2^(exp - 64 L),  N = sum_l limbs[l] 2^(64 l),  L = ceil(prec/64)
 *   nonzero: top bit of limbs[L-1] set, the low 64L-prec bits zero; |exp| <= 2^61
 *   zero:    all limbs zero (sign and exp ignored on input; written as +0, exp 0)
 *   Matrices are row-major with leading dimension ld (entries); limbs are entry-major
 *   (entry e's limbs at limbs[e*L .. e*L+L-1]).  No NaN / Inf encoding exists.
 *
 * Ownership: the caller owns A, B and C (DEVICE memory for mpcgemm/mpcgemm_ex/
 * mpcgemm_rho_bounds; HOST memory for mpcgemm_host).  The library never frees them and
 * owns only its workspace (a per-device grow-only cache released by mpcgemm_release(),
 * or caller memory via opts->workspace).  C must not overlap A or B.  Calls are
 * stream-ordered on opts->stream (NULL: the legacy default stream); A and B must stay
 * unchanged until the stream passes the call.  The host blocks only to read back the
 * 24-byte pre-pass result when slices == 0 (auto).
 *
 * Errors: return 0 = OK, > 0 warning, < 0 error.  No exceptions, no abort, no printing.
 * On an error detected before launch C is untouched; after a CUDA error C is undefined
 * and mpcgemm_last_error() describes it (thread-local).
 */
#ifndef MPCGEMM_H
#define MPCGEMM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MPCGEMM_OK                  0
#define MPCGEMM_ERR_ARG            -1   /* null pointer, m/n/k < 0, ld < cols, bad method      */
#define MPCGEMM_ERR_PREC           -2   /* prec outside [2, 4096]                              */
#define MPCGEMM_ERR_EXP_RANGE      -3   /* |exp| > 2^61 (validate mode)                        */
#define MPCGEMM_ERR_NOT_NORMALIZED -4   /* nonzero mantissa without top bit / low bits set     */
#define MPCGEMM_ERR_ALIAS          -5   /* C overlaps A or B                                   */
#define MPCGEMM_ERR_NOMEM          -6   /* workspace allocation failed / too small             */
#define MPCGEMM_ERR_CUDA           -7   /* CUDA runtime error (see mpcgemm_last_error)         */
#define MPCGEMM_ERR_SLICES         -8   /* forced or derived slice count outside [1, 1024]     */

typedef struct {
    uint8_t  *sign;   /* [rows*ld]      0 = +, 1 = -                                          */
    int64_t  *exp;    /* [rows*ld]      MPFR exponent: |x| in [2^(exp-1), 2^exp)              */
    uint64_t *limbs;  /* [rows*ld*L]    little-endian limbs, entry-major                      */
    int64_t   ld;     /* leading dimension in entries, >= cols                                */
} mpc_rmat;

typedef struct { mpc_rmat re, im; } mpc_cmat;   /* planar complex, one prec for all parts   */

typedef enum { MPCGEMM_3M = 3, MPCGEMM_4M = 4 } mpcgemm_method;

typedef struct {
    void    *stream;          /* cudaStream_t; NULL = legacy default stream                   */
    int32_t  slices;          /* 0 = auto (pre-pass + slice rule); > 0 forces s               */
    int32_t  validate;        /* 1 = check normalization / exponent range on device first      */
    void    *workspace;       /* NULL = library-managed per-device cache                       */
    size_t   workspace_bytes; /* size of caller workspace (>= mpcgemm_workspace_size)          */
    int32_t  timing;          /* 1 = time each stage with CUDA events on opts->stream (the call
                                 then synchronizes the stream before returning)              */
    int32_t  beta;            /* 0: C := alpha A B.  1: C := C + alpha A B -- C is read as input
                                 (in place) and the exact sum is rounded once (SURVEY NEXT-2:
                                 the LU trailing update A22 - L21 U12)      */
    int32_t  alpha_neg;       /* 1: alpha = -1, else alpha = +1                                 */
    int32_t  carrier;         /* slice carrier: 0 = INT8 digits on tcgen05 (default);
                                 1 = the paper's binary64 slices, b = 53 - ceil((53 +
                                 ceil(log2 k)) / 2) bits, on FP64 DMMA (SURVEY
                                 NEXT-1; beta / alpha_neg not supported there)                  */
    int32_t  adaptive;        /* NEXT-4 ("set the optimal number of divisions"):
                                 1 = a certified slice count per block of 256 rows of A / C.
                                 Block b gets s_b = the slice rule applied to the pre-pass over
                                 its rows (against all of B); the digits are split once with
                                 s = max_b s_b and block b uses the TOP s_b digits of every
                                 expansion with Algorithm 2's triangle d = s_b, value
                                 P 2^(eA_i + eB_j + 6 - 8(s_b+1)).  Same error bound per block;
                                 bit-identical to oracle orc_cgemm_ozaki_rows.  Ignored when
                                 slices > 0; INT8 carrier only.  0 = one s for all rows.        */
    int32_t *block_slices;    /* optional HOST output, ceil(m/256) entries: the s used by each
                                 256-row block (all equal to s unless adaptive)               */
    int32_t  device_rule;     /* 1 (with slices == 0): the slice rule runs ON THE DEVICE -- the
                                 pre-pass integers are reduced and the certified s chosen by a
                                 kernel, which selects one of the plans the host prepared for every
                                 s the first pre-pass stage can yield, s_lo = rule(log2 rho = 0) ..
                                 s_hi = rule(minT = 1); the split, slice GEMM and fold read the
                                 chosen plan from device memory.  The call never synchronizes the
                                 host (after the first call of a shape: plans and workspace are
                                 cached), so it can be captured in a CUDA graph.  Same result as
                                 the host rule, bit for bit.  If the certified s falls outside
                                 [s_lo, s_hi] (only when the max-plus stage is needed) nothing is
                                 written to C and mpcgemm_device_rule_result() returns
                                 MPCGEMM_ERR_SLICES -- callers then repeat the call with
                                 device_rule = 0.  Ignored with slices > 0, validate, beta,
                                 alpha_neg, adaptive, carrier = 1; rep->slices is 0 (unknown).    */
} mpcgemm_opts;

typedef struct {
    int32_t slices;           /* s used                                                        */
    int32_t certified;        /* 1 if s came from the certified rule or was forced             */
    int64_t minT, minT1, maxD2;   /* pre-pass integers (-1 when not computed)                  */
    double  log2_rho_hat;     /* the rule's log2 rho-hat                                       */
    int64_t mma_instructions; /* tcgen05.mma count issued by the slice GEMM (K=32 each)         */
    int64_t work_units;       /* slice-GEMM work units (tile, diagonal, chunk, product)         */
    int32_t kernel_launches;  /* kernels this call launched (memsets/copies excluded)           */
    int32_t slice_bits;       /* digit width b: 8 (INT8 carrier) or the binary64 slice width   */
    int32_t slicegemm_ctas;   /* grid of the slice-GEMM launch                                 */
    float   ms_linemax, ms_prepass, ms_split, ms_gemm, ms_fold;   /* opts->timing only         */
    int32_t slices_min;       /* smallest per-block s (== slices unless opts->adaptive)        */
    int32_t partial_slots;    /* int32 partial planes per output element read by the fold       */
    int32_t tile_m, tile_n;   /* output tile of one slice-GEMM work unit (rows x columns)      */
    int64_t mma_issued;       /* tcgen05.mma instructions (K = 32) counted ON THE DEVICE by the
                                 issuing thread of every slice-GEMM CTA (pre-pass T GEMM
                                 excluded); opts->timing only, else -1.  Closed form for a full
                                 triangle: R P ceil(m/tile_m) ceil(n/tile_n) ceil(k/32),
                                 R = 3 (3M) / 4 (4M), P = s (s+1) / 2                          */
} mpcgemm_report;

/* C := A B (auto slice count).  Device pointers.  m, n, k >= 0 (empty: nothing written for
 * m*n == 0; k == 0 writes zeros).  2 <= prec <= 4096. */
int mpcgemm(int64_t m, int64_t n, int64_t k, int32_t prec,
            const mpc_cmat *A, const mpc_cmat *B, mpc_cmat *C, mpcgemm_method method);

/* as mpcgemm, with options (stream, forced slice count, workspace) and an optional report. */
int mpcgemm_ex(int64_t m, int64_t n, int64_t k, int32_t prec,
               const mpc_cmat *A, const mpc_cmat *B, mpc_cmat *C, mpcgemm_method method,
               const mpcgemm_opts *opts, mpcgemm_report *rep);

/* End-to-end call on HOST buffers: copies A and B to the device, computes, copies C back
 * (all inside the call; blocks until C is on the host).  Host pointers; pinned memory
 * recommended.  Uses the library workspace cache plus a device staging cache. */
int mpcgemm_host(int64_t m, int64_t n, int64_t k, int32_t prec,
                 const mpc_cmat *A, const mpc_cmat *B, mpc_cmat *C, mpcgemm_method method,
                 const mpcgemm_opts *opts, mpcgemm_report *rep);

/* Pipelined form of mpcgemm_host for a stream of independent products: same arguments and
 * result, but returns once the call's device work is queued (it blocks only for its own
 * slice-count pre-pass).  The H2D of the inputs runs on a library copy stream into one of two
 * device staging sets, so call i+1's copies overlap call i's slice GEMM, and C's D2H overlaps
 * the next call's compute.  The host buffers A, B, C must stay valid and unmodified until
 * mpcgemm_host_wait() returns; the report is filled at return (opts->timing makes the call
 * synchronize per stage).  Errors detected while queuing are returned by the call (after
 * draining its queued work); asynchronous device faults by mpcgemm_host_wait(). */
int mpcgemm_host_async(int64_t m, int64_t n, int64_t k, int32_t prec,
                       const mpc_cmat *A, const mpc_cmat *B, mpc_cmat *C, mpcgemm_method method,
                       const mpcgemm_opts *opts, mpcgemm_report *rep);

/* Blocks until every mpcgemm_host_async call issued on this device has finished (C on the
 * host).  0 or MPCGEMM_ERR_CUDA. */
int mpcgemm_host_wait(void);

/* The rho-hat pre-pass on this process's A rows:
 *   out[0] = minT  = min_ij T_ij, T = t u (INT8 GEMM), over nonzero rows/columns with
 *                    (|A||B|)_ij != 0  (-1: no such pair)
 *   out[1] = minT1, out[2] = maxD2: the second stage (exact max-plus exponent bound),
 *            computed when out[0] == 0 or full != 0; otherwise out[1] = out[0], out[2] = -1.
 * Multi-GPU: ranks all-reduce MIN of out[0]; if the result is 0 every rank calls again with
 * full = 1 and ranks all-reduce MIN out[1] (ignoring -1) and MAX out[2]; then
 * mpcgemm_slices_for() on the reduced integers gives the common s.  Synchronizes the stream. */
int mpcgemm_rho_bounds(int64_t m, int64_t n, int64_t k, int32_t prec,
                       const mpc_cmat *A, const mpc_cmat *B, int32_t full,
                       const mpcgemm_opts *opts, int64_t out[3]);

/* The slice-count rule:  log2rho = log2(k) + 14 - log2(minT) (minT > 0), or the max of that
 * with minT1 and log2(k) + 2 + maxD2 (minT == 0), or 0 (minT < 0);
 * s = min{ s >= 1 : 8 s >= prec - 4 + log2(c s) + log2rho + 0.1 }, c = 3 (4M), 4 (3M).
 * Returns s, or MPCGEMM_ERR_SLICES if s > 1024. */
int mpcgemm_slices_for(int32_t prec, mpcgemm_method method, int64_t k,
                       int64_t minT, int64_t minT1, int64_t maxD2);

/* Device workspace bytes for one call with s slices (slices <= 0: the s the rule picks at
 * minT = 1, the largest first-stage s for this prec and k -- an auto-s call whose inputs need
 * the max-plus stage may pick more and then runs in row groups).  A smaller caller workspace (or less free
 * device memory, or the MPCGEMM_WS_LIMIT environment variable, bytes) makes the call run in row
 * groups of 256 * 2^j rows (B split once; bit-identical result); ERR_NOMEM only when one
 * 256-row group does not fit. */
size_t mpcgemm_workspace_size(int64_t m, int64_t n, int64_t k, int32_t prec,
                              mpcgemm_method method, int32_t slices);

/* ------------------------------------------------------------------ NEXT-3: complex LU
 * The paper's second workload (Eq. 7, Fig. 3).  All pointers DEVICE; A is
 * n x n (ld >= n), factored in place: P A = L U with L unit lower (strictly below the
 * diagonal) and U upper; ipiv[c] (int64) = the row swapped with row c at step c.  For each
 * panel j0 = 0, K, 2K, ... of width w = min(K, n - j0):
 *   (a) c = j0 .. j0+w-1: pivot p = first argmax_{r >= c} key(A_rc) (key: |re| + |im| as
 *       (max exponent, binary64 sum of the top-53-bit parts) -- DESIGN.md NEXT-3); swap rows c
 *       and p over all n columns; A_rc := cmul(A_rc, crecip(A_cc)) for r > c; A_rt :=
 *       cfms(A_rt, A_rc, A_ct) for r > c, c < t < j0 + w        (LAPACK xGETF2 on the panel)
 *   (b) A_rt := cfms(A_rt, A_rc, A_ct) for c in the panel, c < r < j0 + w, t >= j0 + w
 *                                                                 (U12 := L11^-1 A12)
 *   (c) A22 := A22 - L21 U12 by mpcgemm_ex (method, certified auto s, beta = 1, alpha_neg = 1:
 *       one rounding per element; opts->adaptive passes through)
 * Scalar ops, each real part the exact value rounded once (RNE) to prec:
 *   cmul(x, y) = RNE(x y);  cfms(a, x, y) = RNE(a - x y);  crecip(z) = RNE(conj(z) / |z|^2).
 * Bit-identical to oracle orc_clu_factor.  K = 1 is column-wise LU with rank-1 Ozaki updates;
 * K >= n is unblocked (no GEMM).  2 <= prec <= 1024.  A zero pivot does not stop the
 * factorization; rep->info = c + 1 for the first one (0: nonsingular).  opts: stream,
 * timing (per-phase times; synchronizes), adaptive.  Synchronizes the stream (info readback). */
typedef struct {
    int32_t info;             /* 0, or c + 1 of the first zero pivot                           */
    int32_t gemm_calls;       /* trailing updates through the Ozaki GEMM                       */
    int32_t slices_max;       /* largest slice count of the updates                            */
    int32_t kernel_launches;  /* kernels launched (panel + trsm + GEMM)                        */
    float   ms_panel, ms_trsm, ms_gemm;   /* opts->timing only                                  */
} mpclu_report;

int mpclu_factor(int64_t n, int32_t prec, mpc_cmat *A, int64_t *ipiv, int32_t K, mpcgemm_method method,
                 const mpcgemm_opts *opts, mpclu_report *rep);

/* Eq. 7: B (n x nrhs, ld >= nrhs, DEVICE) := A^-1 B with the factors of mpclu_factor: the row
 * swaps ipiv[0..n) in order; forward B_r := cfms(B_r, L_rc, B_c) (r > c, c ascending);
 * backward B_c := cmul(B_c, crecip(U_cc)), then B_r := cfms(B_r, U_rc, B_c) (r < c, c
 * descending).  2 n + 3 launches (one per substitution step, the reciprocals 1/U_cc all at
 * once first); stream-ordered.  A zero U_cc gives a zero solution row (no error). */
int mpclu_solve(int64_t n, int64_t nrhs, int32_t prec, const mpc_cmat *LU, const int64_t *ipiv, mpc_cmat *B,
                const mpcgemm_opts *opts);

/* Elementwise device MP scalar operations on 1 x cnt DEVICE matrices (used by the tests to
 * check the LU's arithmetic against the oracle): op 0: O = cmul(X, Y); 1: O = cfms(A, X, Y);
 * 2: O = crecip(X) (X != 0); 3: kv[2t] = key exponent, kv[2t+1] = key value (binary64 bits).
 * stream: cudaStream_t (NULL: legacy default stream). */
int mpc_scalar(int32_t op, int64_t cnt, int32_t prec, const mpc_cmat *A, const mpc_cmat *X, const mpc_cmat *Y,
               mpc_cmat *O, int64_t *kv, void *stream);

/* Result of the last device_rule call of shape m x n on this device: synchronizes `stream`
 * (cudaStream_t, NULL = legacy default) and reads the device state.  out[0] = the certified s,
 * out[1..3] = the reduced pre-pass integers (minT, minT1, maxD2).  Returns 0, or
 * MPCGEMM_ERR_SLICES when that s was outside the planned range (C untouched). */
int mpcgemm_device_rule_result(int64_t m, int64_t n, void *stream, int64_t out[4]);

const char *mpcgemm_strerror(int code);
const char *mpcgemm_last_error(void);   /* thread-local detail of the last error              */
void mpcgemm_release(void);              /* frees the cached workspace of the current device   */
int  mpcgemm_version(void);              /* ABI version (100 * major + minor)                  */

#ifdef __cplusplus
}
#endif
#endif /* MPCGEMM_H */
