// kernels.h -- launchers of the sm_100a kernels (internal; the C ABI is include/mpcgemm.h)
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "common.cuh"

namespace mpc {

// Programmatic dependent launch (device-rule calls, set for the call by gemm_impl): the hot-path
// kernels are launched with programmatic stream serialization and each executes
// griddepcontrol.wait (pdl_wait) before touching global memory, so a kernel's launch and
// scheduling overlap its predecessor's tail -- the fixed per-launch cost of tiny calls.
extern thread_local int g_pdl;
template <typename... Exp, typename... Act>
inline cudaError_t launch_pdl(void (*kern)(Exp...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Act &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid; cfg.blockDim = block; cfg.dynamicSmemBytes = smem; cfg.stream = st;
    cudaLaunchAttribute at[1];
    if (g_pdl) {
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
    }
    return cudaLaunchKernelEx(&cfg, kern, static_cast<Act &&>(args)...);
}

struct SliceGemmLaunch {
    GemmParams P;
    const int8_t *digA, *digB;   // [partsA*s][rowsA][kp], [partsB*s][rowsB][kp]
    int64_t rowsA, rowsB, kp;
    int grid;                    // CTAs (tcgen05 path)
    int BM;                      // 128 (one CTA per tile) or 256 (CTA pair, cta_group::2)
    int BN;                      // 128 or 256
    int simt;                    // 1: dp4a cross-check kernel
    int nunits;
    const WorkUnit *units_flat;
};
cudaError_t slicegemm_launch(const SliceGemmLaunch &L, cudaStream_t st);

// a-1: per-line max exponent over nonzero entries of (re, im); side 0 = rows, 1 = columns
cudaError_t linemax_launch(DMat re, DMat im, int64_t rows, int64_t cols, int L, int prec, int side,
                           int64_t *eline, uint8_t *nz, uint32_t *errflag, int validate, cudaStream_t st);

// a-1 for both operands in one scan launch (eAB = eA[m] then eB[n], nzAB likewise)
cudaError_t linemax2_launch(DMat Are, DMat Aim, DMat Bre, DMat Bim, int64_t m, int64_t n, int64_t k, int L, int prec,
                            int64_t *eAB, uint8_t *nzAB, uint32_t *errflag, int validate, cudaStream_t st,
                            int *nlaunch = nullptr, unsigned long long *acc_clean = nullptr, uint8_t *tb = nullptr,
                            int64_t tbkp = 0);
cudaError_t prepass_planes2_launch(DMat Are, DMat Aim, DMat Bre, DMat Bim, int64_t m, int64_t n, int64_t k, int64_t kp,
                                   int L, const int64_t *eA, const int64_t *eB, int8_t *tA, int32_t *relA, int8_t *tB,
                                   int32_t *relB, cudaStream_t st, unsigned long long *fill0 = nullptr,
                                   int64_t nfill0 = 0, unsigned long long *fill1 = nullptr, int64_t nfill1 = 0,
                                   const uint8_t *tb = nullptr);

// a-3: balanced radix-256 digit planes dig[part][alpha][lines][kp]
cudaError_t split_launch(DMat re, DMat im, int side, int64_t lines, int64_t k, int64_t kp, int L,
                         const int64_t *eline, int s, int nparts, int8_t *dig, cudaStream_t st,
                         const DevRuleState *drs = nullptr);

// a-3 for both operands (B then A) in one launch where the TMA split applies
cudaError_t split2_launch(DMat Are, DMat Aim, DMat Bre, DMat Bim, int64_t m, int64_t n, int64_t k, int64_t kp, int L,
                          const int64_t *eA, const int64_t *eB, int s, int nparts, int8_t *digA, int8_t *digB,
                          cudaStream_t st, const DevRuleState *drs = nullptr, int *nlaunch = nullptr);

// 3-D TMA map over the fold's int32 partial planes (slicegemm.cu): box = one row's 256-column strip
// of 8 consecutive slots
int encode_partials_map(void *map, const int32_t *base, int64_t gslots, int slots_per_box);

// 3-D TMA map over ABI limbs (implemented in slicegemm.cu; map = CUtensorMap*, 64-byte aligned)
int encode_limb_map(void *map, const uint64_t *base, int L, uint64_t d1, uint64_t d2, uint64_t stride1,
                    uint64_t stride2, int b1, int b2);

// a-2: pre-pass planes: t[lines][kp] int8 and relative entry exponents rel[lines][kp] int32
cudaError_t prepass_planes_launch(DMat re, DMat im, int side, int64_t lines, int64_t k, int64_t kp, int L,
                                  const int64_t *eline, int8_t *t, int32_t *rel, cudaStream_t st);

// a-2: stage 1 (out_min = min T over nonzero line pairs) and stage 2 (out_min, out_min1,
// out_max2), each an array over the 256-row blocks of A (kSBlk)
// small device -> host results (pre-pass integers, flags) written by SM stores into mapped
// pinned host memory: no copy engine, so they never queue behind a bulk D2H on another stream
cudaError_t readback_launch(void *dst_mapped, const void *src, size_t bytes, cudaStream_t st);
// device-rule mode: stage 2 only if some block's stage-1 minimum is 0 (decided on the device;
// out_*2 arrays, initialised to all-ones), then the slice rule over the reduced integers picks
// the plan (plans[s - s_lo] for s in [s_lo, s_hi]) into *drs
cudaError_t prepass_small_t_launch(const int8_t *tA, const int8_t *tB, int64_t m, int64_t n, int64_t k, int64_t kp,
                                   const uint8_t *nzA, const uint8_t *nzB, int32_t *T, int64_t nstrips,
                                   unsigned long long *min1, cudaStream_t st);
cudaError_t prepass_rule_launch(const int32_t *T, int nslots, int64_t nstrips, int64_t m, int64_t n, int64_t k,
                                int64_t kp, const uint8_t *nzA, const uint8_t *nzB, const int32_t *relA,
                                const int32_t *relB, const unsigned long long *min1, unsigned long long *min2,
                                unsigned long long *min12, long long *max22, int prec, int method,
                                const DevPlan *plans, int s_lo, int s_hi, DevRuleState *drs, cudaStream_t st);
cudaError_t prepass_reduce_launch(const int32_t *T, int nslots, int64_t nstrips,
                                  int64_t m, int64_t n, int64_t k, int64_t kp,
                                  const uint8_t *nzA, const uint8_t *nzB, const int32_t *relA, const int32_t *relB,
                                  int stage, unsigned long long *out_min, unsigned long long *out_min1,
                                  long long *out_max2, cudaStream_t st);

struct FoldParams {
    const int32_t *partials;     // part_off layout
    int64_t nslots, nstrips;
    int64_t m, n;
    int32_t s, method, prec, L;
    const int32_t *slotinfo;     // [(job*(s+2) + r)*2 + {0 base, 1 count}]
    const int64_t *eA, *eB;
    DMatOut Cre, Cim;
    int32_t beta, alpha_neg;     // NEXT-2: C = beta C0 + (-1)^alpha_neg A B (one rounding)
    DMat C0re, C0im;             // may alias Cre / Cim
    const int32_t *sblk;         // NEXT-4: slice count of each 256-row block (<= s), or nullptr
    uint64_t *fix;               // fixed-point scratch, fold_scratch_words(m, ldF, s, L, beta) words
    int64_t ldF;                 // scratch row pitch (a multiple of kFoldLdAlign, >= n)
    const DevRuleState *drs;     // or null; else s, nslots, slotinfo come from drs->cur (F.s: the
                                 // largest candidate s, which sizes shared memory and the scratch)
    int32_t uni1;                // every (job, diagonal) of the plan has exactly one chunk
    int32_t unic;                // 3 jobs with equal chunk counts per diagonal (slots in groups of 3)
    int32_t norm_generic;        // (cross-check) round through the generic local-memory path
    int32_t l2hint;              // partial loads evict-first, fixed-point scratch stores evict-last
};
constexpr int kFoldLdAlign = 4;  // scratch pitch: a multiple of every fold variant's outputs per thread
size_t fold_scratch_words(int64_t m, int64_t ldF, int s, int L, bool beta);
// a-5 + a-6: exact fold (chunk sums, Eq. 5/6 combination, carry) and RNE normalization
cudaError_t fold_normalize_launch(const FoldParams &F, cudaStream_t st);

cudaError_t zero_output_launch(DMatOut C, int64_t m, int64_t n, int L, cudaStream_t st);

// NEXT-1: binary64 slice carrier on FP64 DMMA (fp64path.cu)
cudaError_t split_f64_launch(DMat re, DMat im, int side, int64_t lines, int64_t k, int64_t kp, int L,
                             const int64_t *eline, int s, int b, int nparts, double *dig, cudaStream_t st);
cudaError_t dmma_slicegemm_launch(const double *digA, const double *digB, int64_t m, int64_t n, int64_t kp, int s,
                                  const int4 *units, int nunits, const JobDesc *jobs, int njobs, int64_t *partials,
                                  cudaStream_t st);
cudaError_t fold_f64_launch(const int64_t *partials, int64_t m, int64_t n, int s, int b, int method, int prec, int L,
                            const int64_t *eA, const int64_t *eB, DMatOut Cre, DMatOut Cim, cudaStream_t st);

// NEXT-3: complex LU (lu.cu).  L = limbs per element (1..16).
struct LuScratch { uint8_t *sign; int64_t *exp; uint64_t *limbs; };   // 2 elements (1 / pivot)
cudaError_t lu_pivot_launch(int L, DMatOut re, DMatOut im, int64_t n, int64_t c, int64_t *ipiv, cudaStream_t st);
cudaError_t lu_swap_launch(int L, DMatOut re, DMatOut im, int64_t ncols, int64_t c, const int64_t *ipiv, cudaStream_t st);
cudaError_t lu_recip_launch(int L, DMatOut re, DMatOut im, int64_t c, int prec, LuScratch s, int32_t *info,
                            cudaStream_t st);
cudaError_t lu_scale_launch(int L, DMatOut re, DMatOut im, int64_t r0, int64_t r1, int64_t c, int prec, LuScratch s,
                            cudaStream_t st);
// 1 / A_cc into s (and *info) and A_rc := cmul(A_rc, 1 / A_cc) for r in [r0, r1): one launch when
// the warp kernels apply, else lu_recip_launch + lu_scale_launch
cudaError_t lu_recip_scale_launch(int L, DMatOut re, DMatOut im, int64_t r0, int64_t r1, int64_t c, int prec,
                                  LuScratch s, int32_t *info, int *nlaunch, cudaStream_t st);
cudaError_t lu_update_launch(int L, DMatOut re, DMatOut im, int64_t r0, int64_t r1, int64_t t0, int64_t t1, int64_t c,
                             int prec, cudaStream_t st);
struct SolveScratch {
    DMatOut rre, rim;            // 1 x n: 1 / U_cc
    DMatOut xre, xim;            // n x nrhs: the permuted right-hand sides, then the solution rows
    int64_t *perm;               // n: the row permutation P
};
cudaError_t lu_solve_launch(int L, DMatOut fre, DMatOut fim, int64_t n, const int64_t *ipiv, DMatOut bre, DMatOut bim,
                            int64_t nrhs, int prec, SolveScratch s, cudaStream_t st);
cudaError_t mp_scalar_launch(int L, int op, int64_t cnt, int prec, DMatOut Ar, DMatOut Ai, DMatOut Xr, DMatOut Xi,
                             DMatOut Yr, DMatOut Yi, DMatOut Or, DMatOut Oi, int64_t *kv, cudaStream_t st);

}  // namespace mpc
