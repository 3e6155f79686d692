// common.cuh -- shared declarations of the sm_100a CUDA path (no oracle code here).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define MPC_DEV __device__ __forceinline__

namespace mpc {

constexpr int kMaxSlices = 1024;     // s limit (prec <= 4096 plus exponent spread)
constexpr int kMaxJobs = 3;          // 3M: T1,T2,T3 ; 4M: T1,T2,T34
constexpr int kMaxPairs = 2;         // operand pairs concatenated into one job (4M T34)
// INT32 exactness of one accumulation chunk: |d_p d_q| <= 2^14, so K' <= 131071 products;
// in k-blocks of 128: 1023 blocks = 130944 products.
constexpr int kMaxKBlocksPerChunk = 1023;
constexpr int kBK = 128;             // k-block: 128 int8 = one 128-byte swizzle row
// NEXT-4 (per-block slice counts): the pre-pass reduces, and the adaptive mode chooses s, per
// block of 256 rows of A / C (the CTA-pair tile height)
constexpr int kSBlkShift = 8;
constexpr int kSBlk = 1 << kSBlkShift;

// Device view of one real MP matrix in the ABI format (include/mpcgemm.h).
struct DMat {
    const uint8_t *sign;
    const int64_t *exp;
    const uint64_t *limbs;
    int64_t ld;
};

struct DMatOut {
    uint8_t *sign;
    int64_t *exp;
    uint64_t *limbs;
    int64_t ld;
};

// One slice-GEMM work unit on output tile (tm, tn) of job `job` (job_g = job | G << 8):
//  G = 1: one chunk of anti-diagonal r -- the k-blocks g in [a, b) of the job's concatenated
//         sequence (pair, p = 1..r-1, kb) -- into partial plane slot0;
//  G = 2: anti-diagonals r and r+1 together over the k-blocks kb in [a, b) of every pair and
//         every p, into planes slot0 (D_r) and slot1 (D_{r+1}); each A_p / B_q tile is
//         loaded once and feeds both diagonals.
//  G = 3: anti-diagonal r alone over the k-blocks kb in [a, b) of every pair (a pair segment
//         cut at r = s_b + 1 by a NEXT-4 per-block slice count), into slot0.
struct WorkUnit {
    int32_t job_g, tm, tn, r, a, b, slot0, slot1;
};
__host__ __device__ __forceinline__ int unit_job(const WorkUnit &w) { return w.job_g & 0xFF; }
__host__ __device__ __forceinline__ int unit_G(const WorkUnit &w) { return (w.job_g >> 8) & 0xFF; }
// serpentine k order: units of alternate diagonal pairs walk their k-blocks downward, so a group
// starts on the k-blocks the previous group (the neighbouring diagonals) read last -- still in L2
__host__ __device__ __forceinline__ bool unit_rev(const WorkUnit &w) { return (w.job_g >> 16) & 1; }
__host__ __device__ __forceinline__ int unit_kb(const WorkUnit &w, int i) { return unit_rev(w) ? w.b - 1 - i : w.a + i; }
// p-blocking of a G >= 2 unit: its planes p = 1 .. np (np = r for G = 2, r - 1 for G = 3) are
// walked in nblk blocks, each over all its k-blocks, so one k-block step touches pblk planes
__host__ __device__ __forceinline__ int unit_nblk(int np, int pblk) { return pblk > 0 && np > pblk ? (np + pblk - 1) / pblk : 1; }
__host__ __device__ __forceinline__ int unit_pfirst(int np, int nblk, int j) { return j * np / nblk + 1; }
// job-wide k-phase mode (GemmParams.kmode == 2): the hint of a G >= 2 unit is shared by every
// unit of its (job, k-block chunk) class (id in job_g bits 17..30), and its p-blocks start at
// absolute plane numbers 1, pblk + 1, 2 pblk + 1, ... (the last block takes the remainder), so
// co-running units of neighbouring diagonal pairs walk the same A_p tiles at the same time
__host__ __device__ __forceinline__ int unit_hint(const WorkUnit &w) { return (w.job_g >> 17) & 0x3FFF; }
constexpr int kHintNB = 1024;   // p-block stride of a class-wide position (pair, p-block, k-block)
// tile-wide k-phase mode (GemmParams.kmode == 3, with the tile-major unit order MPCGEMM_ORDER=3):
// the hint (id in job_g bits 17..30) is shared by every unit of one (job, output tile) -- all its
// diagonal pairs and exactness chunks -- and holds the absolute position (pair * kHintNB + p-block)
// * KB + k-block, so the ~74 co-running units of a tile read the same A_p tile at the same time
// and B planes two steps apart (tools/l2sim.cpp: DRAM operand reads ~90 -> ~46 GB at config 4)
__host__ __device__ __forceinline__ int unit_nblk_m(int np, int pblk, int kmode) {
    if (kmode < 2) return unit_nblk(np, pblk);
    return pblk > 0 && np > pblk ? (np + pblk / 2) / pblk : 1;
}
__host__ __device__ __forceinline__ int unit_pfirst_m(int np, int nblk, int j, int pblk, int kmode) {
    if (kmode < 2) return unit_pfirst(np, nblk, j);
    return j >= nblk ? np + 1 : j * pblk + 1;
}

struct JobDesc {
    int32_t npairs;
    int32_t pa[kMaxPairs];   // A-side digit part of each pair (0 Re, 1 Im, 2 Re+Im)
    int32_t pb[kMaxPairs];   // B-side digit part
};

// int32 partial planes, tile-blocked: [128-row block][256-column strip][slot][128][256].  One
// GEMM unit writes one contiguous 128 KB block (write locality); the fold's 128 blocks of one
// (row block, strip) run together and stream every slot block.  Slots are numbered in the
// fold's consumption order (r = s+1..2, job, chunk).
constexpr int kStrip = 256;
constexpr int kRowBlk = 128;
constexpr int64_t kTileElems = (int64_t)kRowBlk * kStrip;
__host__ __device__ __forceinline__ int64_t part_off(int64_t row, int64_t col, int64_t slot, int64_t nslots,
                                                     int64_t nstrips) {
    return (((row >> 7) * nstrips + (col >> 8)) * nslots + slot) * kTileElems + (row & (kRowBlk - 1)) * kStrip +
           (col & (kStrip - 1));
}

// Device-rule mode (opts->device_rule): the slice count is chosen on the device from the pre-pass
// integers, among candidate plans built by the host for every s the first stage can yield; the
// kernels after the rule read the chosen plan from device memory (no host readback).
struct DevPlan {
    const WorkUnit *units;     // the plan's unit list
    int32_t *hot;              // its k-phase hints
    const int32_t *slotinfo;   // its (job, r) -> (first slot, chunk count) table
    int32_t s, nunits, nslots, pad;
};
struct DevRuleState {
    DevPlan cur;               // the chosen plan
    int32_t status;            // 0: ok; MPCGEMM_ERR_SLICES (-8): the certified s is outside the planned
                               // range -- every kernel after the rule returns without writing C
    int32_t s_needed;          // the certified s (also when outside the range)
    int64_t minT, minT1, maxD2;   // the reduced pre-pass integers the rule used
};

struct GemmParams {
    const WorkUnit *units;     // global order: size-descending, tiles of one (job, r, chunk) contiguous
    int32_t nunits;
    int32_t *counter;          // dynamic scheduler: next unit (zeroed before each launch)
    int32_t *partials;         // part_off layout
    int64_t nslots;            // partial planes
    int64_t nstrips;           // ceil(n / 256)
    int32_t m, n;
    int32_t s;                 // slices
    int32_t KB;                // k-blocks per digit plane row
    int32_t partsA, partsB;    // number of digit parts stored per side
    int32_t dbg;               // power experiments only (MPCGEMM_DBG, results invalid when != 0):
                               // bit 0: epilogue skips the partial-plane stores; bit 1: every TMA
                               // load reads plane 0 / tile (0, 0) (L2-resident operands); bit 2: loads
                               // cycle through 8 planes x 2 k-blocks x 2 tiles (~1 MB, varying data);
                               // bit 3: after the first ring fill no loads at all (smem reused)
    int32_t *hot;              // k-phase hints, one per (job, r, chunk) group (or null): the position
                               // (pair, p-block, k-block) a running unit of the group last started;
                               // a new unit of the group begins there (CTA-pair kernel, G >= 2)
    int32_t pblk;              // p-block length of the CTA-pair kernel's G >= 2 units (0: one block)
    int32_t kmode;             // k-phase hint mode: 1 one hint per (job, r, chunk) group; 2 one per
                               // (job, chunk) class with absolute p-blocks (unit_hint); 3 one per
                               // (job, output tile) holding an absolute k-block
    int32_t kk_last;           // K = 32 MMA steps of the last k-block (1..3; 0: all 4): the zero
                               // padding of k up to a multiple of 128 is not multiplied
    unsigned long long *mma_count;   // or null: tcgen05.mma instructions issued, added at CTA exit
    const DevRuleState *drs;         // or null; else s, nunits, nslots, units, hot come from drs->cur
    int32_t halfn;                   // CTA-pair kernel: N = 128 MMAs on a last tile column of <= 128 columns
    JobDesc jobs[kMaxJobs];
};

MPC_DEV uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---------------------------------------------------------------- mbarrier
MPC_DEV void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
MPC_DEV void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
MPC_DEV void mbar_arrive(uint64_t *bar) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar)) : "memory");
}
MPC_DEV void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}"
                 ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
MPC_DEV bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 1000000;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    return ok != 0;
}
// Waits for the phase with the given parity; traps after ~20 s so that a pipeline bug ends
// the kernel with an error instead of hanging the GPU.
MPC_DEV void mbar_wait(uint64_t *bar, uint32_t parity) {
    if (mbar_try_wait(bar, parity)) return;
    const long long t0 = clock64();
    while (!mbar_try_wait(bar, parity)) {
        if (clock64() - t0 > 40000000000ll) __trap();
    }
}

// ---------------------------------------------------------------- clusters (CTA pairs)
MPC_DEV uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
MPC_DEV void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same smem offset in CTA `rank` of the cluster
MPC_DEV uint32_t mapa_rank(uint32_t local_addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_addr), "r"(rank));
    return r;
}
MPC_DEV void mbar_arrive_remote(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// dynamic scheduler: the next unit index, or -1 when the list is done.  Every fetching CTA takes
// exactly one index >= nunits (its last), so the fetch that returns nunits + nfetch - 1 is the
// launch's final access to the counter: it re-arms the counter for the next launch in stream order
// (no memset node before each slice GEMM; the plan zeroes the counter once when it is created)
MPC_DEV int fetch_unit(int32_t *counter, int nunits, int nfetch) {
    const int u = atomicAdd(counter, 1);
    if (u < nunits) return u;
    if (u == nunits + nfetch - 1) atomicExch(counter, 0);
    return -1;
}
MPC_DEV int32_t ld_relaxed_s32(const int32_t *p) {
    int32_t v;
    asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
MPC_DEV void st_relaxed_s32(int32_t *p, int32_t v) {
    asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
MPC_DEV void st_remote_u32(uint32_t cluster_addr, uint32_t v) {
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(cluster_addr), "r"(v) : "memory");
}
// acquire-side wait that also orders remote (cluster-scope) writes
MPC_DEV bool mbar_try_wait_cluster(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2, 1000000;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    return ok != 0;
}
MPC_DEV void mbar_wait_cluster(uint64_t *bar, uint32_t parity) {
    if (mbar_try_wait_cluster(bar, parity)) return;
    const long long t0 = clock64();
    while (!mbar_try_wait_cluster(bar, parity)) {
        if (clock64() - t0 > 40000000000ll) __trap();
    }
}

// ---------------------------------------------------------------- TMA
MPC_DEV void tma_prefetch(const void *tmap) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(tmap) : "memory");
}
MPC_DEV void tma_load_3d(void *dst, const void *tmap, uint64_t *bar, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];"
        ::"r"(smem_u32(dst)), "l"(tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2) : "memory");
}

MPC_DEV void tma_load_3d_hint(void *dst, const void *tmap, uint64_t *bar, int c0, int c1, int c2, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4, %5}], [%2], %6;"
        ::"r"(smem_u32(dst)), "l"(tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "l"(pol) : "memory");
}

// 1-D bulk copy global -> shared, completion counted on an mbarrier (bytes % 16 == 0)
MPC_DEV void bulk_load(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// orders this thread's generic-proxy shared-memory accesses before later async-proxy accesses
// (TMA / bulk copies) -- e.g. before releasing a ring slot that a TMA load will overwrite
// programmatic dependent launch: wait until the preceding grid in the stream has completed and its
// memory is visible (a no-op when the kernel was not launched with programmatic serialization)
MPC_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
MPC_DEV void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// L2 cache policies (createpolicy) and a 16-byte store carrying one
MPC_DEV uint64_t l2_policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
MPC_DEV uint64_t l2_policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
MPC_DEV uint64_t l2_policy_evict_normal() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}
MPC_DEV void st_global_v2u64_hint(void *ptr, uint64_t a, uint64_t b, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v2.u64 [%0], {%1, %2}, %3;" ::"l"(ptr), "l"(a), "l"(b), "l"(pol) : "memory");
}
MPC_DEV void st_global_u64_hint(void *ptr, uint64_t a, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.u64 [%0], %1, %2;" ::"l"(ptr), "l"(a), "l"(pol) : "memory");
}
MPC_DEV void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
MPC_DEV void ld_shared_v4(uint32_t addr, uint32_t &a, uint32_t &b, uint32_t &c, uint32_t &d) {
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "r"(addr) : "memory");
}
MPC_DEV void st_global_v4_hint(void *ptr, int a, int b, int c, int d, uint64_t pol) {
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.s32 [%0], {%1, %2, %3, %4}, %5;"
                 ::"l"(ptr), "r"(a), "r"(b), "r"(c), "r"(d), "l"(pol) : "memory");
}

// 2-SM TMA: both CTAs of a pair load into their own smem; completion bytes are counted on
// the even (leader) CTA's mbarrier (peer bit 24 of the shared::cluster address cleared)
MPC_DEV void tma_load_3d_2sm(void *dst, const void *tmap, uint64_t *bar, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];"
        ::"r"(smem_u32(dst)), "l"(tmap), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1), "r"(c2) : "memory");
}

// ---------------------------------------------------------------- tcgen05
MPC_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
MPC_DEV void tc_fence_after()  { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

template <int NCOLS>
MPC_DEV void tmem_alloc(uint32_t *dst_smem) {   // whole warp
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(smem_u32(dst_smem)), "n"(NCOLS) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <int NCOLS>
MPC_DEV void tmem_alloc_2sm(uint32_t *dst_smem) {   // one warp in each CTA of the pair
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(smem_u32(dst_smem)), "n"(NCOLS) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
template <int NCOLS>
MPC_DEV void tmem_dealloc_2sm(uint32_t taddr) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(NCOLS) : "memory");
}
template <int NCOLS>
MPC_DEV void tmem_dealloc(uint32_t taddr) {     // whole warp
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(NCOLS) : "memory");
}

// D[tmem] (+)= A[smem] * B[smem]^T, signed int8 -> int32, K = 32
MPC_DEV void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate) : "memory");
}
// pair MMA (leader CTA only): D[tmem, both CTAs] (+)= A[smem, 128 rows per CTA] * B[smem, N/2 per CTA]^T
MPC_DEV void mma_i8_2sm(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate) : "memory");
}
// commit the leader's prior MMAs to the mbarrier at the same offset in both CTAs of the pair
MPC_DEV void mma_commit_2sm(uint64_t *bar) {
    asm volatile("{\n\t.reg .b16 msk;\n\tmov.b16 msk, 3;\n\t"
                 "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], msk;\n\t}"
                 ::"r"(smem_u32(bar)) : "memory");
}
MPC_DEV void mma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                 ::"r"(smem_u32(bar)) : "memory");
}

// 32 lanes x 32 columns of 32-bit: thread t of the warp gets row (lane base + t), 32 cols
MPC_DEV void tmem_ld_32x32b_x32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr) : "memory");
}
MPC_DEV void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// Shared-memory matrix descriptor (tcgen05 "matrix descriptor"): K-major operand tile of
// rows x 128 bytes written by TMA with 128-byte swizzle; 8-row core groups 1024 B apart.
//   bits  0-13 start address >> 4     bits 16-29 leading byte offset >> 4 (unused: 1)
//   bits 32-45 stride byte offset >> 4 (1024 B)   bits 46-47 version = 1 (sm_100)
//   bits 49-51 base offset = 0        bits 61-63 layout = 2 (SWIZZLE_128B)
MPC_DEV uint64_t make_sw128_desc(uint32_t smem_addr) {
    uint64_t d = 0;
    d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}

// Instruction descriptor, kind::i8: D = S32 (bits 4-5 = 2), A and B signed 8-bit
// (bits 7-9 = 1, 10-12 = 1), both K-major (bits 15, 16 = 0), N >> 3 at 17-22, M >> 4 at 24-28.
__host__ __device__ constexpr uint32_t make_idesc_i8(int M, int N) {
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

}  // namespace mpc
