// slicegemm.cu -- the triangle of slice products of Algorithm 2 on the
// sm_100a INT8 tensor cores.
//
// Anti-diagonal form of the triangle beta <= d - alpha + 1:  for r = 2..s+1
//     D_r = sum_{alpha + beta = r} A_alpha B_beta        (int32, exact: DESIGN.md "Exactness")
// is computed per output tile and written to int32 partial planes; the fold kernel sums them
// with weights 256^(s+1-r).  Work units (common.cuh) are either one chunk of one diagonal
// (G = 1) or a pair of adjacent diagonals (G = 2) sharing every operand tile:
//     step p = 1..r:  load A_p, B_{r+1-p};  D_{r+1} += A_p B_{r+1-p};  D_r += A_{p-1} B_{r+1-p}
// so each 48 KB stage feeds 8 MMAs instead of 4 (half the L2 / HBM bytes per MMA).
//
// Kernel structure (one CTA per SM, persistent; units from a global atomic counter in a
// locality-friendly order):
//   warp 0 lane 0 : scheduler + TMA producer, STAGES-deep ring of (A 128x128 B, B BNx128 B)
//   warp 1        : TMEM allocator; lane 0 issues tcgen05.mma.cta_group::1.kind::i8
//                   (M = 128, N = BN, K = 32; 4 per 128-byte k-block) into two BN-column
//                   accumulators (D_r at column 0, D_{r+1} at column BN)
//   warps 4..7    : epilogue, tcgen05.ld 32x32b -> registers -> int32 partial planes
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include "common.cuh"
#include "kernels.h"

namespace mpc {

constexpr int kBM = 128;

// The K = 32 MMAs of one stage into accumulator d: unpredicated for a full k-block (a per-MMA
// predicate there cost ~6 % of the tensor pipe's issue rate), guarded for the last, partial one.
// acc0: enable-input of the first MMA (0 overwrites the accumulator).
template <bool PAIR>
MPC_DEV void issue_kblock(uint32_t d, uint32_t a, uint32_t b, uint32_t idesc, uint32_t acc0, int n, uint64_t &cnt) {
    cnt += (uint64_t)n;
    if (n == kBK / 32) {
#pragma unroll
        for (int kk = 0; kk < kBK / 32; kk++) {
            if constexpr (PAIR) mma_i8_2sm(d, make_sw128_desc(a + kk * 32), make_sw128_desc(b + kk * 32), idesc, kk ? 1u : acc0);
            else                mma_i8(d, make_sw128_desc(a + kk * 32), make_sw128_desc(b + kk * 32), idesc, kk ? 1u : acc0);
        }
    } else {
#pragma unroll
        for (int kk = 0; kk < kBK / 32; kk++)
            if (kk < n) {
                if constexpr (PAIR) mma_i8_2sm(d, make_sw128_desc(a + kk * 32), make_sw128_desc(b + kk * 32), idesc, kk ? 1u : acc0);
                else                mma_i8(d, make_sw128_desc(a + kk * 32), make_sw128_desc(b + kk * 32), idesc, kk ? 1u : acc0);
            }
    }
}

template <int BN, int STAGES>
struct TcCfg {
    static constexpr int A_BYTES = kBM * kBK;
    static constexpr int B_BYTES = BN * kBK;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int TMEM_COLS = 2 * BN;           // two accumulators
    static constexpr int QN = 8;                       // unit-index queue depth
    static constexpr int EPI_PITCH = 144;              // epilogue transpose rows (32 int32 + pad)
    static constexpr int EPI_BYTES = 4 * 32 * EPI_PITCH;
    static constexpr size_t SMEM = 1024 /*align slack*/ + (size_t)STAGES * STAGE_BYTES + 512 /*barriers, queue*/ + EPI_BYTES;
};

// digit planes of step (pair, p, kb) of a unit
struct StepPlanes { int planeA, planeB, kb; };

template <int BN, int STAGES>
__global__ void __launch_bounds__(256, 1)
slicegemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ GemmParams P)
{
    pdl_wait();
    using Cfg = TcCfg<BN, STAGES>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *sA = smem;
    uint8_t *sB = smem + STAGES * Cfg::A_BYTES;
    uint64_t *full = reinterpret_cast<uint64_t *>(sB + STAGES * Cfg::B_BYTES);
    uint64_t *empty = full + STAGES;
    uint64_t *tfull = empty + STAGES;                 // accumulators ready (MMA -> epilogue)
    uint64_t *tempty = tfull + 1;                     // accumulators drained (epilogue -> MMA)
    uint64_t *qfull = tempty + 1;                     // unit-index queue (producer -> MMA, epilogue)
    uint64_t *qempty = qfull + Cfg::QN;
    int32_t *uq = reinterpret_cast<int32_t *>(qempty + Cfg::QN);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(uq + Cfg::QN);
    uint8_t *skk = reinterpret_cast<uint8_t *>(tmem_slot + 1);   // per stage: MMA K-steps to issue
    uint8_t *sE = smem + (size_t)STAGES * Cfg::STAGE_BYTES + 512;   // epilogue transposes [warp][32][pitch]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (P.drs && P.drs->status != 0) return;          // device rule: s outside the planned range
    const DevPlan *dp = P.drs ? &P.drs->cur : nullptr;
    const WorkUnit *units = dp ? dp->units : P.units;
    const int nunits = dp ? dp->nunits : P.nunits;
    const int64_t nslots = dp ? dp->nslots : P.nslots;
    if (warp == 0 && lane == 0) {
        for (int i = 0; i < STAGES; i++) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
        mbar_init(tfull, 1);
        mbar_init(tempty, 128);
        for (int i = 0; i < Cfg::QN; i++) { mbar_init(&qfull[i], 1); mbar_init(&qempty[i], 1 + 4); }
        fence_barrier_init();
        tma_prefetch(&tmA);
        tma_prefetch(&tmB);
    }
    if (warp == 1) tmem_alloc<Cfg::TMEM_COLS>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const int s = dp ? dp->s : P.s, KB = P.KB;

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- scheduler + TMA producer: units are taken in list order from a
            // global counter, so co-running CTAs work on neighbouring tiles of the same
            // (job, r, chunk) and share the digit-plane tiles in L2
            int stage = 0; uint32_t phase = 0;
            int qs = 0; uint32_t qph = 0;
            auto load = [&](int planeA, int planeB, int kb, int tm, int tn) {
                mbar_wait(&empty[stage], phase ^ 1);
                skk[stage] = (uint8_t)(kb == KB - 1 && P.kk_last ? P.kk_last : kBK / 32);   // before the arrive (release)
                mbar_arrive_expect_tx(&full[stage], Cfg::STAGE_BYTES);
                tma_load_3d(sA + stage * Cfg::A_BYTES, &tmA, &full[stage], kb * kBK, tm * kBM, planeA);
                tma_load_3d(sB + stage * Cfg::B_BYTES, &tmB, &full[stage], kb * kBK, tn * BN, planeB);
                if (++stage == STAGES) { stage = 0; phase ^= 1; }
            };
            for (;;) {
                int u = fetch_unit(P.counter, nunits, (int)gridDim.x);
                mbar_wait(&qempty[qs], qph ^ 1);
                *reinterpret_cast<volatile int32_t *>(&uq[qs]) = u;
                mbar_arrive(&qfull[qs]);
                if (++qs == Cfg::QN) { qs = 0; qph ^= 1; }
                if (u < 0) break;
                const WorkUnit w = units[u];
                const JobDesc &J = P.jobs[unit_job(w)];
                if (unit_G(w) == 2) {
                    for (int pr = 0; pr < J.npairs; pr++)
                        for (int i = 0; i < w.b - w.a; i++)
                            for (int p = 1; p <= w.r; p++)          // A_p, B_{r+1-p}
                                load(J.pa[pr] * s + p - 1, J.pb[pr] * s + (w.r - p), unit_kb(w, i), w.tm, w.tn);
                } else if (unit_G(w) == 3) {                        // D_r alone over kb in [a, b)
                    for (int pr = 0; pr < J.npairs; pr++)
                        for (int i = 0; i < w.b - w.a; i++)
                            for (int p = 1; p < w.r; p++)           // A_p, B_{r-p}
                                load(J.pa[pr] * s + p - 1, J.pb[pr] * s + (w.r - p - 1), unit_kb(w, i), w.tm, w.tn);
                } else {
                    const int per_pair = (w.r - 1) * KB;
                    for (int g = w.a; g < w.b; g++) {
                        const int pair = g / per_pair;
                        const int rem = g - pair * per_pair;
                        const int p0 = rem / KB;                    // alpha - 1
                        const int kb = rem - p0 * KB;
                        load(J.pa[pair] * s + p0, J.pb[pair] * s + (w.r - 2 - p0), kb, w.tm, w.tn);
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (lane == 0) {
            // ---------------- MMA issuer
            constexpr uint32_t idesc = make_idesc_i8(kBM, BN);
            const uint32_t d0 = tmem_base, d1 = tmem_base + (uint32_t)BN;
            int stage = 0; uint32_t phase = 0;
            uint32_t tphase = 0;
            int qs = 0; uint32_t qph = 0;
            uint64_t nmma = 0;                                // MMA instructions issued (P.mma_count)
            for (;;) {
                mbar_wait(&qfull[qs], qph);
                const int u = *reinterpret_cast<volatile int32_t *>(&uq[qs]);
                mbar_arrive(&qempty[qs]);
                if (++qs == Cfg::QN) { qs = 0; qph ^= 1; }
                if (u < 0) { if (P.mma_count) atomicAdd(P.mma_count, (unsigned long long)nmma); break; }
                const WorkUnit w = units[u];
                const JobDesc &J = P.jobs[unit_job(w)];
                mbar_wait(tempty, tphase ^ 1);
                tc_fence_after();
                if (unit_G(w) == 2) {
                    int prev = 0;
                    for (int pr = 0; pr < J.npairs; pr++)
                        for (int i = 0; i < w.b - w.a; i++)
                            for (int p = 1; p <= w.r; p++) {
                                mbar_wait(&full[stage], phase);
                                tc_fence_after();
                                const uint32_t a0 = smem_u32(sA + stage * Cfg::A_BYTES);
                                const uint32_t b0 = smem_u32(sB + stage * Cfg::B_BYTES);
                                const bool first = (pr == 0 && i == 0);
                                const int nkk = (unit_kb(w, i) == KB - 1 && P.kk_last) ? P.kk_last : kBK / 32;
                                issue_kblock<false>(d1, a0, b0, idesc, (first && p == 1) ? 0u : 1u, nkk, nmma);   // D_{r+1} += A_p B_{r+1-p}
                                if (p >= 2) {                           // D_r += A_{p-1} B_{r+1-p}
                                    issue_kblock<false>(d0, smem_u32(sA + prev * Cfg::A_BYTES), b0, idesc,
                                                        (first && p == 2) ? 0u : 1u, nkk, nmma);
                                    mma_commit(&empty[prev]);           // A_{p-1} no longer needed
                                }
                                if (p == w.r) mma_commit(&empty[stage]);   // A_r pairs only with B_1
                                prev = stage;
                                if (++stage == STAGES) { stage = 0; phase ^= 1; }
                            }
                } else {
                    const int nsteps = unit_G(w) == 3 ? J.npairs * (w.b - w.a) * (w.r - 1) : w.b - w.a;
                    for (int g = 0; g < nsteps; g++) {
                        mbar_wait(&full[stage], phase);
                        tc_fence_after();
                        const uint32_t a0 = smem_u32(sA + stage * Cfg::A_BYTES);
                        const uint32_t b0 = smem_u32(sB + stage * Cfg::B_BYTES);
                        issue_kblock<false>(d0, a0, b0, idesc, g > 0 ? 1u : 0u, skk[stage], nmma);
                        mma_commit(&empty[stage]);
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                    }
                }
                mma_commit(tfull);                            // accumulators ready
                tphase ^= 1;
            }
        }
        __syncwarp();
    } else if (warp >= 4) {
        // ---------------- epilogue: TMEM -> registers -> int32 partial planes
        const int q = warp & 3;                               // TMEM lane quarter of this warp
        const uint64_t pol = l2_policy_evict_first();         // partials: streaming, keep operands in L2
        uint32_t tphase = 0;
        int qs = 0; uint32_t qph = 0;
        for (;;) {
            mbar_wait(&qfull[qs], qph);
            const int u = *reinterpret_cast<volatile int32_t *>(&uq[qs]);
            __syncwarp();
            if (lane == 0) mbar_arrive(&qempty[qs]);
            if (++qs == Cfg::QN) { qs = 0; qph ^= 1; }
            if (u < 0) break;
            const WorkUnit w = units[u];
            mbar_wait(tfull, tphase);
            tc_fence_after();
            // (as the CTA-pair kernel: 32 x 32 blocks through a padded shared-memory transpose, a
            // warp store = 4 whole 128-byte row segments; four TMEM loads per wait)
            const int row0 = w.tm * kBM + q * 32;
            const uint32_t swa = smem_u32(sE) + (uint32_t)(q * 32 * Cfg::EPI_PITCH);
            const int rsub = lane >> 3, piece = lane & 7;
            for (int acc = 0; acc < (unit_G(w) == 2 ? 2 : 1); acc++) {
                const int64_t slot = acc ? w.slot1 : w.slot0;
#pragma unroll 1
                for (int c0 = 0; c0 < BN / 32; c0 += 4) {
                    uint32_t v[4][32];
#pragma unroll
                    for (int j = 0; j < 4; j++)
                        tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + (c0 + j) * 32), v[j]);
                    tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < 4; j++) {
#pragma unroll
                        for (int g4 = 0; g4 < 8; g4++)
                            st_shared_v4(swa + (uint32_t)(lane * Cfg::EPI_PITCH + 16 * g4), v[j][4 * g4], v[j][4 * g4 + 1],
                                         v[j][4 * g4 + 2], v[j][4 * g4 + 3]);
                        __syncwarp();
                        // 32 columns inside one 256-column strip
                        int32_t *out = P.partials + part_off(row0, w.tn * BN + (c0 + j) * 32, slot, nslots, P.nstrips) + 4 * piece;
#pragma unroll
                        for (int g = 0; g < 8; g++) {
                            const int rr = 4 * g + rsub;
                            uint32_t x0, x1, x2, x3;
                            ld_shared_v4(swa + (uint32_t)(rr * Cfg::EPI_PITCH + 16 * piece), x0, x1, x2, x3);
                            if (row0 + rr < P.m)
                                st_global_v4_hint(out + (int64_t)rr * kStrip, (int)x0, (int)x1, (int)x2, (int)x3, pol);
                        }
                        __syncwarp();
                    }
                }
            }
            tc_fence_before();
            mbar_arrive(tempty);
            tphase ^= 1;
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) tmem_dealloc<Cfg::TMEM_COLS>(tmem_base);
}

// ------------------------------------------------------------------ CTA-pair (cta_group::2) kernel
// Same work units on 256 x 256 output tiles computed by a CTA pair: each CTA loads its 128 rows
// of the A tile and its 128 rows of the B tile (32 KB per stage instead of 48 KB), the even CTA
// issues tcgen05.mma.cta_group::2 (M = 256, N = 256) and each CTA's TMEM holds its 128 rows of
// both accumulators.  The even CTA schedules units and forwards each index to its peer.
template <int STAGES>
struct Tc2Cfg {
    static constexpr int BN = 256;                     // pair tile 256 x 256
    static constexpr int A_BYTES = 128 * kBK;          // this CTA's half of the A tile
    static constexpr int B_BYTES = 128 * kBK;          // this CTA's half of the B tile
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int TMEM_COLS = 512;
    static constexpr int QN = 8;
    static constexpr int EPI_PITCH = 144;              // epilogue transpose rows (32 int32 + pad)
    static constexpr int EPI_BYTES = 4 * 32 * EPI_PITCH;
    static constexpr size_t SMEM = 1024 + (size_t)STAGES * STAGE_BYTES + 512 + EPI_BYTES;
};

template <int STAGES>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1)
slicegemm_tc2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ GemmParams P)
{
    pdl_wait();
    using Cfg = Tc2Cfg<STAGES>;
    constexpr int BN = Cfg::BN;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *sA = smem;
    uint8_t *sB = smem + STAGES * Cfg::A_BYTES;
    uint64_t *full = reinterpret_cast<uint64_t *>(sB + STAGES * Cfg::B_BYTES);   // leader's used
    uint64_t *empty = full + STAGES;                  // both CTAs (multicast commit)
    uint64_t *tfull = empty + STAGES;                 // both CTAs (multicast commit)
    uint64_t *tempty = tfull + 1;                     // leader's used: 2 x 128 epilogue arrivals
    uint64_t *qfull = tempty + 1;                     // both CTAs (leader producer arrives on both)
    uint64_t *qempty = qfull + Cfg::QN;               // leader's used: 10 arrivals
    int32_t *uq = reinterpret_cast<int32_t *>(qempty + Cfg::QN);
    int32_t *uqr = uq + Cfg::QN;                      // each unit's k-phase rotation (both producers)
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(uqr + Cfg::QN);
    uint8_t *skk = reinterpret_cast<uint8_t *>(tmem_slot + 1);   // per stage: MMA K-steps to issue
    uint8_t *sE = smem + (size_t)STAGES * Cfg::STAGE_BYTES + 512;   // epilogue transposes [warp][32][pitch]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (P.drs && P.drs->status != 0) return;          // device rule: s outside the planned range
    const DevPlan *dp = P.drs ? &P.drs->cur : nullptr;
    const WorkUnit *units = dp ? dp->units : P.units;
    const int nunits = dp ? dp->nunits : P.nunits;
    const int64_t nslots = dp ? dp->nslots : P.nslots;
    int32_t *const hot = dp ? dp->hot : P.hot;
    // a tile column with at most 128 valid columns (n mod 256 in (0, 128]): N = 128 MMAs (each CTA
    // supplies 64 B rows), half the epilogue -- instead of multiplying 128 zero-padded columns
    auto half_n = [&](int tn) { return P.halfn && P.n - tn * 256 <= 128; };
    const uint32_t rank = cluster_ctarank();
    if (warp == 0 && lane == 0) {
        for (int i = 0; i < STAGES; i++) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
        mbar_init(tfull, 1);
        mbar_init(tempty, 2 * 128);
        for (int i = 0; i < Cfg::QN; i++) { mbar_init(&qfull[i], 1); mbar_init(&qempty[i], 1 + 4 + 1 + 4); }
        fence_barrier_init();
        tma_prefetch(&tmA);
        tma_prefetch(&tmB);
    }
    if (warp == 1) tmem_alloc_2sm<Cfg::TMEM_COLS>(tmem_slot);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const uint32_t lead_qempty = mapa_rank(smem_u32(qempty), 0);
    const uint32_t lead_tempty = mapa_rank(smem_u32(tempty), 0);
    const uint32_t peer_uq = mapa_rank(smem_u32(uq), 1);
    const uint32_t peer_uqr = mapa_rank(smem_u32(uqr), 1);
    const uint32_t peer_qfull = mapa_rank(smem_u32(qfull), 1);
    const int s = dp ? dp->s : P.s, KB = P.KB;

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- (leader) scheduler + both CTAs' TMA producers
            int stage = 0; uint32_t phase = 0;
            int qs = 0; uint32_t qph = 0;
            int nload = 0;
            auto load = [&](int planeA, int planeB, int kb, int tm, int tn, bool a_only = false) {
                mbar_wait(&empty[stage], phase ^ 1);
                skk[stage] = (uint8_t)(kb == KB - 1 && P.kk_last ? P.kk_last : kBK / 32);   // before the arrive (release)
                if ((P.dbg & 8) && nload >= STAGES) {          // experiment: no operand traffic at all
                    if (rank == 0) mbar_arrive(&full[stage]);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                    return;
                }
                nload++;
                if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * (a_only ? Cfg::A_BYTES : Cfg::STAGE_BYTES));
                if (P.dbg & 2) { planeA = planeB = 0; kb = 0; tm = tn = 0; }
                if (P.dbg & 4) { planeA &= 7; planeB &= 7; kb &= 1; tm &= 1; tn &= 1; }   // ~1 MB of varying operands
                tma_load_3d_2sm(sA + stage * Cfg::A_BYTES, &tmA, &full[stage], kb * kBK, tm * 256 + (int)rank * 128, planeA);
                if (!a_only)                                  // (a p-block's lead stage needs only A)
                    tma_load_3d_2sm(sB + stage * Cfg::B_BYTES, &tmB, &full[stage], kb * kBK,
                                    tn * 256 + (int)rank * (half_n(tn) ? 64 : 128), planeB);
                if (++stage == STAGES) { stage = 0; phase ^= 1; }
            };
            for (;;) {
                int u, rot = 0;
                if (rank == 0) {
                    u = fetch_unit(P.counter, nunits, (int)gridDim.x / 2);   // one fetcher per CTA pair
                    if (u >= 0 && hot) {
                        // k-phase alignment: begin at the (pair, k-block) position the group's
                        // running units are on, so the units sharing a digit-plane tile read it
                        // within one k-block step of each other (an L2 hit) whatever their start
                        const WorkUnit &wu = units[u];
                        if (unit_G(wu) >= 2) {
                            const int nkb = wu.b - wu.a, npairs = P.jobs[unit_job(wu)].npairs;
                            const int nblk = unit_nblk_m(unit_G(wu) == 2 ? wu.r : wu.r - 1, P.pblk, P.kmode);
                            const int npos = npairs * nblk * nkb;
                            if (P.kmode == 2) {               // class-wide position -> this unit's
                                const int h = ld_relaxed_s32(hot + unit_hint(wu));
                                const int hk = h % nkb, hb = (h / nkb) % kHintNB, hp = h / (nkb * kHintNB);
                                rot = (h > 0 && hp < npairs && hb < nblk) ? (hp * nblk + hb) * nkb + hk : 0;
                            } else if (P.kmode == 3) {        // tile-wide absolute position
                                const int h = ld_relaxed_s32(hot + unit_hint(wu));
                                const int hk = h % KB, hb = (h / KB) % kHintNB, hp = h / (KB * kHintNB);
                                const int kk = (hk >= wu.a && hk < wu.b) ? hk - wu.a : 0;
                                rot = (hp < npairs && hb < nblk) ? (hp * nblk + hb) * nkb + kk : 0;
                            } else {
                                const int h = ld_relaxed_s32(hot + wu.slot0);
                                rot = (h > 0 && h < npos) ? h : 0;
                            }
                        }
                    }
                    mbar_wait_cluster(&qempty[qs], qph ^ 1);
                    *reinterpret_cast<volatile int32_t *>(&uq[qs]) = u;
                    *reinterpret_cast<volatile int32_t *>(&uqr[qs]) = rot;
                    st_remote_u32(peer_uq + 4 * qs, (uint32_t)u);
                    st_remote_u32(peer_uqr + 4 * qs, (uint32_t)rot);
                    mbar_arrive(&qfull[qs]);
                    mbar_arrive_remote(peer_qfull + 8 * qs);
                } else {
                    mbar_wait_cluster(&qfull[qs], qph);
                    u = *reinterpret_cast<volatile int32_t *>(&uq[qs]);
                    rot = *reinterpret_cast<volatile int32_t *>(&uqr[qs]);
                    mbar_arrive_remote(lead_qempty + 8 * qs);
                }
                if (++qs == Cfg::QN) { qs = 0; qph ^= 1; }
                if (u < 0) break;
                const WorkUnit w = units[u];
                const JobDesc &J = P.jobs[unit_job(w)];
                if (unit_G(w) >= 2) {
                    // positions (pair, p-block, k-block), t = 0 .. npos - 1 taken from rot on; D_r and
                    // D_{r+1} (G = 2: A_p, B_{r+1-p}) or D_r alone (G = 3: A_p, B_{r-p}).  A G = 2
                    // block that starts at p0 > 1 first loads A_{p0-1} (D_r's partner of B_{r+1-p0})
                    const int g2 = unit_G(w) == 2;
                    const int np = g2 ? w.r : w.r - 1, nkb = w.b - w.a, nblk = unit_nblk_m(np, P.pblk, P.kmode);
                    const int npos = J.npairs * nblk * nkb;
                    int pos = rot;
                    for (int t = 0; t < npos; t++) {
                        const int pb = pos / nkb, pr = pb / nblk, blk = pb - pr * nblk;
                        const int kb = unit_kb(w, pos - pb * nkb);
                        const int p0 = unit_pfirst_m(np, nblk, blk, P.pblk, P.kmode);
                        const int p1 = unit_pfirst_m(np, nblk, blk + 1, P.pblk, P.kmode) - 1;
                        if (rank == 0 && hot) {
                            if (P.kmode == 2) st_relaxed_s32(hot + unit_hint(w), (pr * kHintNB + blk) * nkb + (pos - pb * nkb));
                            else if (P.kmode == 3) st_relaxed_s32(hot + unit_hint(w), (pr * kHintNB + blk) * KB + kb);
                            else st_relaxed_s32(hot + w.slot0, pos);
                        }
                        if (g2 && p0 > 1) load(J.pa[pr] * s + p0 - 2, 0, kb, w.tm, w.tn, true);   // A_{p0-1} only
                        for (int p = p0; p <= p1; p++)
                            load(J.pa[pr] * s + p - 1, J.pb[pr] * s + (w.r - p - 1 + g2), kb, w.tm, w.tn);
                        if (++pos == npos) pos = 0;
                    }
                } else {
                    const int per_pair = (w.r - 1) * KB;
                    for (int g = w.a; g < w.b; g++) {
                        const int pair = g / per_pair;
                        const int rem = g - pair * per_pair;
                        const int p0 = rem / KB;
                        const int kb = rem - p0 * KB;
                        load(J.pa[pair] * s + p0, J.pb[pair] * s + (w.r - 2 - p0), kb, w.tm, w.tn);
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (lane == 0 && rank == 0) {
            // ---------------- MMA issuer (leader CTA only)
            constexpr uint32_t idesc_full = make_idesc_i8(256, BN), idesc_half = make_idesc_i8(256, BN / 2);
            const uint32_t d0 = tmem_base, d1 = tmem_base + (uint32_t)BN;
            int stage = 0; uint32_t phase = 0;
            uint32_t tphase = 0;
            int qs = 0; uint32_t qph = 0;
            uint64_t nmma = 0;                                // MMA instructions issued (P.mma_count)
            for (;;) {
                mbar_wait_cluster(&qfull[qs], qph);
                const int u = *reinterpret_cast<volatile int32_t *>(&uq[qs]);
                const int rot = *reinterpret_cast<volatile int32_t *>(&uqr[qs]);
                mbar_arrive(&qempty[qs]);
                if (++qs == Cfg::QN) { qs = 0; qph ^= 1; }
                if (u < 0) { if (P.mma_count) atomicAdd(P.mma_count, (unsigned long long)nmma); break; }
                const WorkUnit w = units[u];
                const JobDesc &J = P.jobs[unit_job(w)];
                const uint32_t idesc = half_n(w.tn) ? idesc_half : idesc_full;   // ragged last tile column: N = 128
                mbar_wait_cluster(tempty, tphase ^ 1);
                tc_fence_after();
                if (unit_G(w) == 2) {
                    // the producer's stage sequence: per position a block p0..p1 (plus the A_{p0-1}
                    // lead stage when p0 > 1); an accumulator's first MMA overwrites it
                    const int nkb = w.b - w.a, nblk = unit_nblk_m(w.r, P.pblk, P.kmode), npos = J.npairs * nblk * nkb;
                    uint32_t acc0 = 0, acc1 = 0;
                    int pos = rot;
                    for (int t = 0; t < npos; t++) {
                        const int blk = (pos / nkb) % nblk;
                        const int p0 = unit_pfirst_m(w.r, nblk, blk, P.pblk, P.kmode);
                        const int p1 = unit_pfirst_m(w.r, nblk, blk + 1, P.pblk, P.kmode) - 1;
                        // MMA K-steps of this position's k-block (from registers: a shared-memory
                        // read here would sit between each stage's barrier and its first MMA)
                        const int nkk = (unit_kb(w, pos % nkb) == KB - 1 && P.kk_last) ? P.kk_last : kBK / 32;
                        int prev = -1;
                        if (p0 > 1) {                                   // lead stage: A_{p0-1}
                            mbar_wait(&full[stage], phase);
                            prev = stage;
                            if (++stage == STAGES) { stage = 0; phase ^= 1; }
                        }
                        for (int p = p0; p <= p1; p++) {
                            mbar_wait(&full[stage], phase);
                            tc_fence_after();
                            const uint32_t a0 = smem_u32(sA + stage * Cfg::A_BYTES);
                            const uint32_t b0 = smem_u32(sB + stage * Cfg::B_BYTES);
                            issue_kblock<true>(d1, a0, b0, idesc, acc1, nkk, nmma);   // D_{r+1} += A_p B_{r+1-p}
                            acc1 = 1u;
                            if (prev >= 0) {                            // D_r += A_{p-1} B_{r+1-p}
                                issue_kblock<true>(d0, smem_u32(sA + prev * Cfg::A_BYTES), b0, idesc, acc0, nkk, nmma);
                                acc0 = 1u;
                                mma_commit_2sm(&empty[prev]);
                            }
                            if (p == p1) mma_commit_2sm(&empty[stage]);
                            prev = stage;
                            if (++stage == STAGES) { stage = 0; phase ^= 1; }
                        }
                        if (++pos == npos) pos = 0;
                    }
                } else {
                    const int nsteps = unit_G(w) == 3 ? J.npairs * (w.b - w.a) * (w.r - 1) : w.b - w.a;
                    for (int g = 0; g < nsteps; g++) {
                        mbar_wait(&full[stage], phase);
                        tc_fence_after();
                        const uint32_t a0 = smem_u32(sA + stage * Cfg::A_BYTES);
                        const uint32_t b0 = smem_u32(sB + stage * Cfg::B_BYTES);
                        issue_kblock<true>(d0, a0, b0, idesc, g > 0 ? 1u : 0u, skk[stage], nmma);
                        mma_commit_2sm(&empty[stage]);
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                    }
                }
                mma_commit_2sm(tfull);                        // both CTAs' accumulators ready
                tphase ^= 1;
            }
        }
        __syncwarp();
    } else if (warp >= 4) {
        // ---------------- epilogue (both CTAs): this CTA's 128 rows of the pair tile
        const int q = warp & 3;
        const uint64_t pol = l2_policy_evict_first();
        uint32_t tphase = 0;
        int qs = 0; uint32_t qph = 0;
        for (;;) {
            mbar_wait_cluster(&qfull[qs], qph);
            const int u = *reinterpret_cast<volatile int32_t *>(&uq[qs]);
            __syncwarp();
            if (lane == 0) {
                if (rank == 0) mbar_arrive(&qempty[qs]);
                else mbar_arrive_remote(lead_qempty + 8 * qs);
            }
            if (++qs == Cfg::QN) { qs = 0; qph ^= 1; }
            if (u < 0) break;
            const WorkUnit w = units[u];
            mbar_wait(tfull, tphase);
            tc_fence_after();
            // TMEM gives lane l row l: a direct store puts 32 rows' 16-byte pieces in one warp store
            // (32 partial-sector writes) -- the drain then held up the next unit's MMAs (both
            // accumulators are in use), e.g. 23 % of config 5's k = 128 GEMMs.  Each 32 x 32 block
            // goes through a padded shared-memory transpose instead, so a warp store writes 4 whole
            // 128-byte row segments; four 32-column TMEM loads are in flight per wait
            const int row0 = w.tm * 256 + (int)rank * 128 + q * 32;        // this warp's first row
            const uint32_t swa = smem_u32(sE) + (uint32_t)(q * 32 * Cfg::EPI_PITCH);
            const int rsub = lane >> 3, piece = lane & 7;
            for (int acc = 0; acc < (unit_G(w) == 2 ? 2 : 1); acc++) {
                const int64_t slot = acc ? w.slot1 : w.slot0;
#pragma unroll 1
                for (int c0 = 0; c0 < (half_n(w.tn) ? BN / 64 : BN / 32); c0 += 4) {
                    uint32_t v[4][32];
#pragma unroll
                    for (int j = 0; j < 4; j++)
                        tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + (c0 + j) * 32), v[j]);
                    tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < 4; j++) {
#pragma unroll
                        for (int g4 = 0; g4 < 8; g4++)
                            st_shared_v4(swa + (uint32_t)(lane * Cfg::EPI_PITCH + 16 * g4), v[j][4 * g4], v[j][4 * g4 + 1],
                                         v[j][4 * g4 + 2], v[j][4 * g4 + 3]);
                        __syncwarp();
                        int32_t *out = P.partials + part_off(row0, w.tn * BN + (c0 + j) * 32, slot, nslots, P.nstrips) + 4 * piece;
#pragma unroll
                        for (int g = 0; g < 8; g++) {
                            const int rr = 4 * g + rsub;
                            uint32_t x0, x1, x2, x3;
                            ld_shared_v4(swa + (uint32_t)(rr * Cfg::EPI_PITCH + 16 * piece), x0, x1, x2, x3);
                            if (!(P.dbg & 1) && row0 + rr < P.m)
                                st_global_v4_hint(out + (int64_t)rr * kStrip, (int)x0, (int)x1, (int)x2, (int)x3, pol);
                        }
                        __syncwarp();
                    }
                }
            }
            tc_fence_before();
            if (rank == 0) mbar_arrive(tempty);
            else mbar_arrive_remote(lead_tempty);
            tphase ^= 1;
        }
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    if (warp == 1) tmem_dealloc_2sm<Cfg::TMEM_COLS>(tmem_base);
}

// ------------------------------------------------------------------ SIMT cross-check kernel
// Same work list and output, computed with dp4a on CUDA cores (used by the tests to check
// the tensor-core kernel bitwise; selected with MPCGEMM_SLICEGEMM_SIMT=1).  One CTA per
// (unit, 32x32 subtile), one thread per 4 output elements of each accumulator.
__global__ void __launch_bounds__(256)
slicegemm_simt_kernel(const int8_t *__restrict__ digA, const int8_t *__restrict__ digB,
                      int64_t rowsA, int64_t rowsB, int64_t kp, const WorkUnit *units, int BM, int BN,
                      const GemmParams P)
{
    __shared__ int32_t sa[32][kBK / 4 + 1];
    __shared__ int32_t sb[32][kBK / 4 + 1];
    const WorkUnit w = units[blockIdx.x];
    const JobDesc &J = P.jobs[unit_job(w)];
    const int G = unit_G(w);
    const int sub = blockIdx.y;                   // 32x32 subtile index within BM x BN
    const int sub_m = sub % (BM / 32), sub_n = sub / (BM / 32);
    const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;   // 32 x 8
    const int64_t row0 = (int64_t)w.tm * BM + sub_m * 32;
    const int64_t col0 = (int64_t)w.tn * BN + sub_n * 32;
    int32_t acc[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
    // enumerate (accumulator, A plane, B plane, kb) exactly as the tensor-core kernel pairs them
    const int npairs = J.npairs;
    const int nsteps = G == 2 ? npairs * (w.b - w.a) * w.r * 2 : G == 3 ? npairs * (w.b - w.a) * (w.r - 1) : (w.b - w.a);
    for (int t = 0; t < nsteps; t++) {
        int which, planeA, planeB, kb;
        if (G == 2) {
            int x = t;
            const int half = x & 1; x >>= 1;          // 0: D_{r+1} (A_p, B_{r+1-p}); 1: D_r (A_p, B_{r-p})
            const int p = x % w.r + 1; x /= w.r;
            kb = w.a + x % (w.b - w.a); x /= (w.b - w.a);
            const int pr = x;
            if (half == 0) { which = 1; planeA = J.pa[pr] * P.s + p - 1; planeB = J.pb[pr] * P.s + (w.r - p); }
            else {
                if (p >= w.r) continue;
                which = 0; planeA = J.pa[pr] * P.s + p - 1; planeB = J.pb[pr] * P.s + (w.r - 1 - p);
            }
        } else if (G == 3) {                          // (pair, kb, p) with p = 1..r-1: D_r only
            int x = t;
            const int p = x % (w.r - 1) + 1; x /= (w.r - 1);
            kb = w.a + x % (w.b - w.a); x /= (w.b - w.a);
            const int pr = x;
            which = 0; planeA = J.pa[pr] * P.s + p - 1; planeB = J.pb[pr] * P.s + (w.r - p - 1);
        } else {
            const int g = w.a + t;
            const int per_pair = (w.r - 1) * P.KB;
            const int pair = g / per_pair;
            const int rem = g - pair * per_pair;
            const int p0 = rem / P.KB;
            kb = rem - p0 * P.KB;
            which = 0; planeA = J.pa[pair] * P.s + p0; planeB = J.pb[pair] * P.s + (w.r - 2 - p0);
        }
        const int8_t *pa = digA + ((int64_t)planeA * rowsA) * kp;
        const int8_t *pb = digB + ((int64_t)planeB * rowsB) * kp;
        __syncthreads();
        for (int q = threadIdx.x; q < 32 * (kBK / 4); q += 256) {
            int rr = q / (kBK / 4), cc = q % (kBK / 4);
            int64_t kk = (int64_t)kb * kBK + cc * 4;
            int32_t va = 0, vb = 0;
            if (row0 + rr < rowsA && kk < kp) va = *reinterpret_cast<const int32_t *>(pa + (row0 + rr) * kp + kk);
            if (col0 + rr < rowsB && kk < kp) vb = *reinterpret_cast<const int32_t *>(pb + (col0 + rr) * kp + kk);
            sa[rr][cc] = va; sb[rr][cc] = vb;
        }
        __syncthreads();
        for (int e = 0; e < 4; e++) {
            const int r_ = ty * 4 + e;
            int32_t v = acc[which][e];
#pragma unroll 8
            for (int cc = 0; cc < kBK / 4; cc++) v = __dp4a(sa[r_][cc], sb[tx][cc], v);
            acc[which][e] = v;
        }
    }
    for (int a = 0; a < (G == 2 ? 2 : 1); a++)
        for (int e = 0; e < 4; e++) {
            const int64_t row = row0 + ty * 4 + e, col = col0 + tx;
            const int slot = a ? w.slot1 : w.slot0;
            // G = 2 keeps D_r in acc[0] and D_{r+1} in acc[1]
            if (row < P.m && col < P.nstrips * kStrip) P.partials[part_off(row, col, slot, P.nslots, P.nstrips)] = acc[a][e];
        }
}

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void *p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// 3-D map over the uint64 limbs of ABI entries for the staged split (stages.cu): dims {L, d1, d2},
// strides (bytes) of dims 1, 2; box {L, b1, b2}; the swizzle matches the 8L-byte rows (L = 16: 128B,
// 8: 64B, 4: 32B, 2: none).  Returns 0 on success.
int encode_limb_map(void *map, const uint64_t *base, int L, uint64_t d1, uint64_t d2, uint64_t stride1,
                    uint64_t stride2, int b1, int b2) {
    auto enc = get_encode();
    if (!enc) return -1;
    CUtensorMapSwizzle sw = L == 16 ? CU_TENSOR_MAP_SWIZZLE_128B : L == 8 ? CU_TENSOR_MAP_SWIZZLE_64B
                          : L == 4 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_NONE;
    cuuint64_t dims[3] = {(cuuint64_t)L, (cuuint64_t)d1, (cuuint64_t)d2};
    cuuint64_t strides[2] = {(cuuint64_t)stride1, (cuuint64_t)stride2};
    cuuint32_t box[3] = {(cuuint32_t)L, (cuuint32_t)b1, (cuuint32_t)b2};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(reinterpret_cast<CUtensorMap *>(map), CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, const_cast<uint64_t *>(base),
                     dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : -2;
}

// 3-D map over the int32 partial planes for the fold's producer: dims {256 columns of a strip,
// 128 rows of a row block, global slot g = (rowblk * nstrips + strip) * nslots + slot}, box
// {256, 1, slots_per_box}: one TMA load brings one row's strip for that many consecutive slots.
// Returns 0 on success.
int encode_partials_map(void *map, const int32_t *base, int64_t gslots, int slots_per_box) {
    auto enc = get_encode();
    if (!enc) return -1;
    cuuint64_t dims[3] = {(cuuint64_t)kStrip, (cuuint64_t)kRowBlk, (cuuint64_t)gslots};
    cuuint64_t strides[2] = {(cuuint64_t)kStrip * 4, (cuuint64_t)kTileElems * 4};
    cuuint32_t box[3] = {(cuuint32_t)kStrip, 1, (cuuint32_t)slots_per_box};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(reinterpret_cast<CUtensorMap *>(map), CU_TENSOR_MAP_DATA_TYPE_INT32, 3, const_cast<int32_t *>(base),
                     dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : -2;
}

// L2 promotion of the digit-plane loads (MPCGEMM_L2PROMO = 0/64/128/256): 128 B = one box row,
// 148 GB DRAM reads per cfg4 launch vs 161 GB with 256 B (same time within noise)
static CUtensorMapL2promotion l2_promotion() {
    const char *e = getenv("MPCGEMM_L2PROMO");
    const int v = e && *e ? atoi(e) : 128;
    return v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE : v == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
         : v == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
}

// 3-D map over digit planes int8 [planes][rows][kp] with box {128, box_rows, 1}, 128B swizzle
static int make_plane_map(CUtensorMap *map, const int8_t *base, int64_t planes, int64_t rows, int64_t kp, int box_rows) {
    auto enc = get_encode();
    if (!enc) return -1;
    cuuint64_t dims[3] = {(cuuint64_t)kp, (cuuint64_t)rows, (cuuint64_t)planes};
    cuuint64_t strides[2] = {(cuuint64_t)kp, (cuuint64_t)(kp * rows)};
    cuuint32_t box[3] = {(cuuint32_t)kBK, (cuuint32_t)box_rows, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t *>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, l2_promotion(),
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : -2;
}

template <int BN, int STAGES>
static cudaError_t launch_tc(const SliceGemmLaunch &L, cudaStream_t st) {
    using Cfg = TcCfg<BN, STAGES>;
    CUtensorMap ta, tb;
    if (make_plane_map(&ta, L.digA, (int64_t)L.P.partsA * L.P.s, L.rowsA, L.kp, kBM)) return cudaErrorInvalidValue;
    if (make_plane_map(&tb, L.digB, (int64_t)L.P.partsB * L.P.s, L.rowsB, L.kp, BN)) return cudaErrorInvalidValue;
    auto kern = slicegemm_tc_kernel<BN, STAGES>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM);
    if (e != cudaSuccess) return e;
    return launch_pdl(kern, dim3(L.grid), dim3(256), Cfg::SMEM, st, ta, tb, L.P);
}

template <int STAGES>
static cudaError_t launch_tc2(const SliceGemmLaunch &L, cudaStream_t st) {
    using Cfg = Tc2Cfg<STAGES>;
    CUtensorMap ta, tb;
    if (make_plane_map(&ta, L.digA, (int64_t)L.P.partsA * L.P.s, L.rowsA, L.kp, 128)) return cudaErrorInvalidValue;
    if (make_plane_map(&tb, L.digB, (int64_t)L.P.partsB * L.P.s, L.rowsB, L.kp, 128)) return cudaErrorInvalidValue;
    auto kern = slicegemm_tc2_kernel<STAGES>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM);
    if (e != cudaSuccess) return e;
    return launch_pdl(kern, dim3(L.grid & ~1), dim3(256), Cfg::SMEM, st, ta, tb, L.P);
}

cudaError_t slicegemm_launch(const SliceGemmLaunch &L, cudaStream_t st) {
    if (L.grid <= 0) return cudaSuccess;
    if (L.simt) {
        dim3 grid(L.nunits, (L.BM / 32) * (L.BN / 32));
        slicegemm_simt_kernel<<<grid, 256, 0, st>>>(L.digA, L.digB, L.rowsA, L.rowsB, L.kp, L.units_flat, L.BM, L.BN, L.P);
        return cudaGetLastError();
    }
    if (L.BM == 256) return launch_tc2<6>(L, st);
    if (L.BN == 256) return launch_tc<256, 4>(L, st);
    if (L.BN == 128) return launch_tc<128, 6>(L, st);
    return cudaErrorInvalidValue;
}

}  // namespace mpc
