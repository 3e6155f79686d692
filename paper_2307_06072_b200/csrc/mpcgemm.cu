// mpcgemm.cu -- host orchestration and the C ABI (include/mpcgemm.h).
//
// One call = the whole hot path of SURVEY.md 8(a), stream-ordered:
//   a-1 linemax (eA, eB)  ->  [a-2 pre-pass: t/u planes, T = t u on the tensor cores,
//   min-reduce, 24-byte readback, optional exact max-plus stage, slice rule]  ->
//   a-3 split (digit planes)  ->  a-4 slice GEMMs (tcgen05 INT8)  ->  a-5/a-6 fold+normalize
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <queue>
#include <string>
#include <tuple>
#include <functional>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/mpcgemm.h"
#include "common.cuh"
#include "kernels.h"
#include "rule.cuh"

namespace mpc { thread_local int g_pdl = 0; }         // kernels.h: launch_pdl
using namespace mpc;

namespace {

thread_local std::string g_last_error;

int fail(int code, const char *what, cudaError_t e = cudaSuccess) {
    g_last_error = what;
    if (e != cudaSuccess) { g_last_error += ": "; g_last_error += cudaGetErrorString(e); }
    return code;
}

#define CK(expr)                                                         \
    do {                                                                 \
        cudaError_t e_ = (expr);                                         \
        if (e_ != cudaSuccess) return fail(MPCGEMM_ERR_CUDA, #expr, e_); \
    } while (0)

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// NVTX range per stage of the hot path (host-side launch sequence; visible in nsys / ncu --nvtx)
struct Nvtx {
    explicit Nvtx(const char *name) { nvtxRangePushA(name); }
    ~Nvtx() { nvtxRangePop(); }
};
int env_int(const char *name, int dflt);
// device rule: the small-shape pre-pass (T by dp4a and the stage-1 minimum in one launch, no T GEMM;
// MPCGEMM_PREPASS_SMALL=0: the tcgen05 T GEMM path)
// a-1 scan -> a-2 planes: the entries' top bytes [2 parts][m + n lines][kp] in the library's dc.tb
// buffer (MPCGEMM_PLANES_TB=0: the planes read the limbs).  (Not in dc.lm: that buffer's first
// 8 (m + n) bytes must stay zero between calls of any shape.)
inline bool planes_tb_on() { return env_int("MPCGEMM_PLANES_TB", 1) != 0; }
inline bool prepass_small(int64_t m, int64_t n, int64_t k) {
    return k > 0 && k <= 65536 && m * n * k <= (int64_t(1) << 27) && env_int("MPCGEMM_PREPASS_SMALL", 1) != 0;
}
// k-phase hint mode of the CTA-pair slice GEMM (MPCGEMM_KPHASE); the tile-wide mode 3 encodes an
// absolute k-block in an int32 position, so it falls back to mode 2 when KB >= 2^20
inline int kphase_mode(int64_t KB) {
    const int m = env_int("MPCGEMM_KPHASE", 2);
    return m == 3 && KB >= (1 << 20) ? 2 : m;
}

// ---------------------------------------------------------------- workspace cache
struct DevCache {
    void *ws = nullptr; size_t ws_bytes = 0;
    void *meta = nullptr; size_t meta_bytes = 0;
    void *stage[2] = {}; size_t stage_bytes[2] = {}; // mpcgemm_host device staging, two sets:
                                                     // an async call fills one while the
                                                     // previous call computes from the other
    int stage_next = 0;
    cudaStream_t h2d_stream = nullptr;               // mpcgemm_host: H2D of the inputs
    cudaEvent_t stage_in[2] = {}, stage_free[2] = {};
    void *rb = nullptr; size_t rb_bytes = 0;         // mapped pinned host memory for readback()
    void *lu = nullptr; size_t lu_bytes = 0;         // NEXT-3 LU scratch (1 / pivot, info)
    void *tb = nullptr; size_t tb_bytes = 0;         // a-1 -> a-2: the entries' top bytes
    void *lm = nullptr; size_t lm_bytes = 0;         // a-1 exponent accumulators + done counter: zero
                                                     // between calls (the scan's last block re-zeroes)
    void *solve = nullptr; size_t solve_bytes = 0;   // NEXT-3 solve scratch (1 / U_cc, X)
    cudaStream_t copy_stream = nullptr;              // mpcgemm_host: D2H of finished row groups
    cudaEvent_t group_event = nullptr;
    cudaEvent_t done = nullptr;                      // completion of the last call's device work
    unsigned long long *mma_dev = nullptr;           // device MMA counter (opts->timing calls)
};

// The cached workspace / scratch of a device is shared by every call, whatever its stream:
// each call's device work is ordered after the previous call's (an event wait on the new
// stream; a no-op on the same stream), so calls on different streams cannot overlap on it.
// Construct with g_mu held; the destructor records this call's completion (g_mu still held).
struct StreamOrder {
    DevCache &dc;
    cudaStream_t st;
    bool capturing = false;                          // inside CUDA graph capture: the graph orders
    StreamOrder(DevCache &d, cudaStream_t s) : dc(d), st(s) {   // its nodes, no cross-stream event
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        cudaStreamIsCapturing(st, &cs);
        capturing = cs != cudaStreamCaptureStatusNone;
        if (dc.done && !capturing) cudaStreamWaitEvent(st, dc.done, 0);
    }
    ~StreamOrder() {
        if (capturing) return;
        if (!dc.done) cudaEventCreateWithFlags(&dc.done, cudaEventDisableTiming);
        cudaEventRecord(dc.done, st);
    }
};
std::mutex g_mu;
std::map<int, DevCache> g_cache;

int grow(void **p, size_t *have, size_t need) {
    if (*have >= need) return 0;
    if (*p) { cudaDeviceSynchronize(); cudaFree(*p); *p = nullptr; *have = 0; }
    size_t sz = align_up(need + (need >> 3), 1 << 20);
    cudaError_t e = cudaMalloc(p, sz);
    if (e != cudaSuccess) { *p = nullptr; cudaGetLastError(); return fail(MPCGEMM_ERR_NOMEM, "cudaMalloc workspace", e); }
    *have = sz;
    return 0;
}

// Stream-ordered read of a few device words to the host (caller holds g_mu): a kernel stores
// them into mapped pinned memory, then the stream is synchronized.  Unlike a D2H memcpy it does
// not wait for the copy engine, which may be busy with a queued call's bulk D2H of C.
int readback(int dev, void *out, const void *src, size_t bytes, cudaStream_t st) {
    DevCache &dc = g_cache[dev];
    if (dc.rb_bytes < bytes) {
        if (dc.rb) { cudaStreamSynchronize(st); cudaFreeHost(dc.rb); dc.rb = nullptr; dc.rb_bytes = 0; }
        const size_t sz = align_up(std::max<size_t>(bytes, 4096), 4096);
        cudaError_t e = cudaHostAlloc(&dc.rb, sz, cudaHostAllocMapped | cudaHostAllocPortable);
        if (e != cudaSuccess) { dc.rb = nullptr; cudaGetLastError(); return fail(MPCGEMM_ERR_NOMEM, "cudaHostAlloc readback", e); }
        dc.rb_bytes = sz;
    }
    void *dptr = nullptr;
    CK(cudaHostGetDevicePointer(&dptr, dc.rb, 0));
    CK(readback_launch(dptr, src, bytes, st));
    CK(cudaStreamSynchronize(st));
    memcpy(out, dc.rb, bytes);
    return 0;
}

// per-device stage events for opts->timing
struct StageEvents {
    cudaEvent_t ev[6] = {};
    bool ok = false;
};
std::map<int, StageEvents> g_events;

StageEvents *stage_events(int dev) {
    StageEvents &E = g_events[dev];
    if (!E.ok) {
        for (auto &e : E.ev) if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
        E.ok = true;
    }
    return &E;
}

// ---------------------------------------------------------------- plans (work lists)
// the fold's group-of-three slot order may be used (MPCGEMM_FOLD_UNIC != 0, no shared-memory-limbs fold)
bool fold_unic_allowed() {
    const char *u = getenv("MPCGEMM_FOLD_UNIC");
    return !(u && atoi(u) == 0) && !getenv("MPCGEMM_FOLD_SFIX");
}

struct PlanKey {
    int64_t m, n, k; int s, method, BM, BN, grid, simt, maxkb, g2, order;
    std::vector<int32_t> sblk;   // NEXT-4: per-256-row-block slice counts (empty: s everywhere)
    int unic_ok = fold_unic_allowed() ? 1 : 0;
    bool operator<(const PlanKey &o) const {
        return std::tie(m, n, k, s, method, BM, BN, grid, simt, maxkb, g2, order, sblk, unic_ok) <
               std::tie(o.m, o.n, o.k, o.s, o.method, o.BM, o.BN, o.grid, o.simt, o.maxkb, o.g2, o.order, o.sblk, o.unic_ok);
    }
};
struct Plan {
    WorkUnit *d_units = nullptr;
    int32_t *d_counter = nullptr;
    int32_t *d_slotinfo = nullptr;
    int nunits = 0, nslots = 0, grid = 0;
    bool uni1 = false;             // every (job, diagonal) has exactly one chunk (3 slots per diagonal)
    bool unic = false;             // 3 jobs and, per diagonal, the same chunk count for every job
    int64_t mma = 0;
    JobDesc jobs[kMaxJobs];
    int njobs = 0, partsA = 0, partsB = 0;
};
std::map<std::pair<int, PlanKey>, Plan> g_plans;

void method_jobs(int method, Plan &P) {
    for (auto &j : P.jobs) { j.npairs = 0; j.pa[0] = j.pa[1] = j.pb[0] = j.pb[1] = 0; }
    if (method == 3) {   // Eq. 6: T1 = ReA ReB, T2 = ImA ImB, T3 = (ReA+ImA)(ReB+ImB)
        P.njobs = 3; P.partsA = P.partsB = 3;
        for (int q = 0; q < 3; q++) { P.jobs[q].npairs = 1; P.jobs[q].pa[0] = q; P.jobs[q].pb[0] = q; }
    } else if (method == 4) {   // Eq. 5: T1 = ReA ReB, T2 = ImA ImB, T34 = ReA ImB + ImA ReB
        P.njobs = 3; P.partsA = P.partsB = 2;
        P.jobs[0].npairs = 1; P.jobs[0].pa[0] = 0; P.jobs[0].pb[0] = 0;
        P.jobs[1].npairs = 1; P.jobs[1].pa[0] = 1; P.jobs[1].pb[0] = 1;
        P.jobs[2].npairs = 2; P.jobs[2].pa[0] = 0; P.jobs[2].pb[0] = 1; P.jobs[2].pa[1] = 1; P.jobs[2].pb[1] = 0;
    } else {             // pre-pass: one job, one pair (t, u), r = 2 only
        P.njobs = 1; P.partsA = P.partsB = 1;
        P.jobs[0].npairs = 1;
    }
}

// Diagonal segments of one job: either a pair (r, r+1) sharing operand tiles (G = 2, the kb
// range cut into nch chunks so that each accumulator sums <= kMaxKBlocksPerChunk k-blocks) or
// a single diagonal r (G = 1, its concatenated (pair, p, kb) sequence cut into nch chunks).
struct Segment { int q, r, G; int64_t nch; };

int64_t exact_cap();

std::vector<Segment> diag_segments(const Plan &P, int64_t KB, int s, int method, int target, bool g2) {
    std::vector<Segment> segs;
    const int rmax = method == 0 ? 2 : s + 1;
    const int64_t cap = exact_cap();
    for (int q = 0; q < P.njobs; q++) {
        const int64_t np = P.jobs[q].npairs;
        int r = 2;
        while (r <= rmax) {
            if (g2 && r + 1 <= rmax && np * r <= cap) {
                // D_{r+1} sums np * r k-blocks per kb: exact if np * r * kbc <= cap
                int64_t kbc = std::min<int64_t>(KB, cap / (np * r));
                kbc = std::max<int64_t>(1, std::min<int64_t>(kbc, target / (np * (2 * r - 1))));
                segs.push_back({q, r, 2, (KB + kbc - 1) / kbc});
                r += 2;
            } else {
                const int64_t G = np * (r - 1) * KB;
                // with pairs, a single diagonal (the odd top one) has about half a pair unit's work:
                // cut it only for exactness, so its slots match the other diagonals' (the fold's
                // pair-entry mode needs one chunk per diagonal wherever exactness allows)
                const int64_t chunk = std::max<int64_t>(1, g2 ? cap : std::min<int64_t>(cap, target));
                segs.push_back({q, r, 1, (G + chunk - 1) / chunk});
                r += 1;
            }
        }
    }
    return segs;
}

bool g2_enabled() { return env_int("MPCGEMM_G2", 1) != 0; }

// Builds the unit list (segments x chunks x output tiles), each unit with its own partial
// planes, and the slot table (job, r) -> (first plane, chunk count) used by the fold.
int build_plan(int dev, const PlanKey &key, Plan **out, cudaStream_t st) {
    auto it = g_plans.find({dev, key});
    if (it != g_plans.end()) { *out = &it->second; return 0; }
    if (g_plans.size() >= 512) {                       // bound the cache (many shapes, e.g. LU updates)
        cudaDeviceSynchronize();                       // queued kernels may still read a plan's units
        for (auto &kv : g_plans) {
            cudaFree(kv.second.d_units); cudaFree(kv.second.d_counter); cudaFree(kv.second.d_slotinfo);
        }
        g_plans.clear();
    }
    Plan P;
    method_jobs(key.method, P);
    const int s = key.s;
    const int64_t KB = (key.k + kBK - 1) / kBK;
    const int64_t tiles_m = (key.m + key.BM - 1) / key.BM, tiles_n = (key.n + key.BN - 1) / key.BN;
    std::vector<int32_t> slotinfo((size_t)kMaxJobs * (s + 2) * 2, 0);
    const std::vector<Segment> segs = diag_segments(P, KB, s, key.method, key.maxkb, key.g2);
    for (const Segment &sg : segs)                     // the fold's chunk-count table is 16-bit
        if (sg.nch > 65535) return fail(MPCGEMM_ERR_ARG, "k too large: more than 65535 exactness chunks per diagonal");
    // slot numbers follow the fold's consumption order: r = s+1 .. 2, job, chunk
    for (const Segment &sg : segs)
        for (int d = 0; d < sg.G; d++) slotinfo[(sg.q * (s + 2) + sg.r + d) * 2 + 1] = (int32_t)sg.nch;
    // slots of one diagonal r: in the order (job, chunk), or -- when the 3 jobs have equal chunk
    // counts on every diagonal (unic) -- (chunk, job), so the fold reads a diagonal as groups of
    // one chunk per job at fixed offsets.  (One chunk everywhere, uni1: both orders coincide.)
    // slotinfo keeps each (job, r)'s first slot (job 0's is the diagonal's first either way)
    int nslots = 0;
    const int rtop = key.method == 0 ? 2 : s + 1;
    auto cnt = [&](int q, int r) { return slotinfo[(q * (s + 2) + r) * 2 + 1]; };
    P.uni1 = P.njobs == 3;
    P.unic = P.njobs == 3 && key.unic_ok;
    for (int r = 2; r <= rtop; r++)
        for (int q = 0; q < P.njobs; q++) {
            P.uni1 = P.uni1 && cnt(q, r) == 1;
            P.unic = P.unic && cnt(q, r) == cnt(0, r);
        }
    std::vector<std::vector<int32_t>> slotid((size_t)P.njobs * (s + 2));
    for (int r = rtop; r >= 2; r--) {
        int maxc = 0;
        for (int q = 0; q < P.njobs; q++) maxc = std::max(maxc, cnt(q, r));
        auto put = [&](int q, int c) {
            if (c == 0) slotinfo[(q * (s + 2) + r) * 2] = nslots;
            slotid[(size_t)q * (s + 2) + r].push_back(nslots++);
        };
        if (P.unic)
            for (int c = 0; c < maxc; c++)
                for (int q = 0; q < P.njobs; q++) put(q, c);
        else
            for (int q = 0; q < P.njobs; q++)
                for (int c = 0; c < cnt(q, r); c++) put(q, c);
    }
    auto slot_of = [&](int q, int r, int64_t c) { return slotid[(size_t)q * (s + 2) + r][(size_t)c]; };
    std::vector<WorkUnit> units;
    // NEXT-4: a row tile of block b takes the segments whose first diagonal r <= sblk[b] + 1; a
    // pair (r, r+1) with r = sblk[b] + 1 becomes a G = 3 unit computing D_r alone
    auto in_tri = [&](int64_t tm, int r) {
        return key.sblk.empty() || r <= key.sblk[(size_t)((tm * key.BM) >> kSBlkShift)] + 1;
    };
    // k-phase mode 2 (job-wide hints): a class id per (job, k-block chunk) in job_g bits 17..30;
    // every unit of a class walks its k-blocks upward (no serpentine), so positions agree
    // k-phase mode 3 (tile-wide hints): one id per (job, output tile), absolute k-blocks
    const int kmode = kphase_mode(KB);
    const bool serp = kmode < 2 && env_int("MPCGEMM_SERPENTINE", 1) != 0;
    std::map<std::tuple<int, int, int>, int32_t> hint_ids;
    int32_t nhint = 0;
    auto hint_tile = [&](int q, int64_t tm, int64_t tn, int32_t a, int32_t b) -> int32_t {
        if (kmode != 3) {
            auto it = hint_ids.emplace(std::make_tuple(q, (int)a, (int)b), (int32_t)hint_ids.size()).first;
            nhint = std::max<int32_t>(nhint, (it->second & 0x3FFF) + 1);
            return (it->second & 0x3FFF) << 17;
        }
        const int32_t id = (int32_t)(((int64_t)q * tiles_m * tiles_n + tm * tiles_n + tn) & 0x3FFF);   // (a shared
        nhint = std::max<int32_t>(nhint, id + 1);      //  id only costs L2 reuse, never exactness)
        return id << 17;
    };
    // K = 32 MMAs per k-block step: 4, except kk_last for the last (zero-padded) k-block
    const int64_t kkl = ((key.k - 1) % kBK) / 32 + 1;
    auto kk_sum = [&](int64_t a, int64_t b) { return (b - a) * (kBK / 32) - ((a <= KB - 1 && KB - 1 < b) ? kBK / 32 - kkl : 0); };
    for (const Segment &sg : segs) {
        const int q = sg.q, r = sg.r;
        const int64_t np = P.jobs[q].npairs;
        if (sg.G == 2) {
            for (int64_t c = 0; c < sg.nch; c++) {
                const int32_t a = (int32_t)(c * KB / sg.nch), b = (int32_t)((c + 1) * KB / sg.nch);
                for (int64_t tm = 0; tm < tiles_m; tm++)
                    for (int64_t tn = 0; tn < tiles_n; tn++) {
                        if (!in_tri(tm, r)) continue;
                        const int32_t rev = serp && ((r >> 1) & 1) ? (1 << 16) : 0;
                        if (!in_tri(tm, r + 1)) {              // block's last diagonal is r: D_r alone
                            units.push_back({q | (3 << 8) | rev | hint_tile(q, tm, tn, a, b), (int32_t)tm, (int32_t)tn, r, a, b, slot_of(q, r, c), -1});
                            P.mma += np * kk_sum(a, b) * (r - 1);
                            continue;
                        }
                        units.push_back({q | (2 << 8) | rev | hint_tile(q, tm, tn, a, b), (int32_t)tm, (int32_t)tn, r, a, b,
                                         slot_of(q, r, c), slot_of(q, r + 1, c)});
                        P.mma += np * kk_sum(a, b) * (2 * r - 1);
                    }
            }
        } else {
            const int64_t G = np * (r - 1) * KB;
            for (int64_t c = 0; c < sg.nch; c++) {
                const int32_t a = (int32_t)(c * G / sg.nch), b = (int32_t)((c + 1) * G / sg.nch);
                for (int64_t tm = 0; tm < tiles_m; tm++)
                    for (int64_t tn = 0; tn < tiles_n; tn++) {
                        if (!in_tri(tm, r)) continue;
                        units.push_back({q | (1 << 8), (int32_t)tm, (int32_t)tn, r, a, b, slot_of(q, r, c), -1});
                        P.mma += (int64_t)(b - a) * (kBK / 32) - (b / KB - a / KB) * (kBK / 32 - kkl);
                    }
            }
        }
    }
    auto work = [&](const WorkUnit &w) -> int64_t {
        const int64_t np = P.jobs[unit_job(w)].npairs;
        return unit_G(w) == 2 ? np * (w.b - w.a) * (2 * w.r - 1)
             : unit_G(w) == 3 ? np * (w.b - w.a) * (w.r - 1) : (int64_t)(w.b - w.a);
    };
    if (key.order == 3) {
        // job-major, then tile-major, then longest first: the ~74 co-running units are all the
        // diagonal pairs (and exactness chunks) of one or two output tiles, so with the tile-wide
        // k-phase hint (KPHASE=3) they read the same A_p tile together and each B plane within a
        // few steps of each other (tools/l2sim.cpp models the operand stream)
        std::stable_sort(units.begin(), units.end(), [&](const WorkUnit &a, const WorkUnit &b) {
            if (unit_job(a) != unit_job(b)) return unit_job(a) < unit_job(b);
            if (a.tm != b.tm) return a.tm < b.tm;
            if (a.tn != b.tn) return a.tn < b.tn;
            return work(a) > work(b);
        });
    } else if (key.order == 2) {
        // job-major; within a job the units of one k-block chunk class (a, b) together -- classes
        // by their smallest unit, largest first, so the job still ends on its smallest units --
        // then longest first: co-running groups are neighbouring diagonal pairs on the SAME
        // k-blocks (with the class-wide k-phase hint they read the same A_p tiles and B planes
        // two steps apart), instead of alternating between the chunks of a multi-chunk diagonal
        std::map<int, int64_t> cmin;                   // class id (G >= 2) -> smallest unit work
        auto cls = [&](const WorkUnit &w) { return unit_G(w) >= 2 ? unit_hint(w) : -1 - unit_job(w); };
        for (const WorkUnit &w : units) {
            auto it = cmin.find(cls(w));
            if (it == cmin.end()) cmin[cls(w)] = work(w); else it->second = std::min(it->second, work(w));
        }
        std::stable_sort(units.begin(), units.end(), [&](const WorkUnit &a, const WorkUnit &b) {
            if (unit_job(a) != unit_job(b)) return unit_job(a) < unit_job(b);
            const int ca = cls(a), cb = cls(b);
            if (ca != cb) {
                const int64_t ma = cmin[ca], mb = cmin[cb];
                if (ma != mb) return ma > mb;
                return ca < cb;
            }
            return work(a) > work(b);
        });
    } else if (key.order == 1) {
        // job-major, then longest first: co-running units are neighbouring diagonal pairs of
        // one job and read mostly the same digit planes; the tail is the last job's smallest
        std::stable_sort(units.begin(), units.end(), [&](const WorkUnit &a, const WorkUnit &b) {
            if (unit_job(a) != unit_job(b)) return unit_job(a) < unit_job(b);
            return work(a) > work(b);
        });
    } else {
        std::stable_sort(units.begin(), units.end(), [&](const WorkUnit &a, const WorkUnit &b) { return work(a) > work(b); });
    }
    int grid = (int)std::min<int64_t>(key.grid, (int64_t)units.size() * (key.BM == 256 ? 2 : 1));
    if (key.BM == 256) grid = std::max(2, grid & ~1);          // CTA pairs
    const std::vector<WorkUnit> &flat = units;
    P.nunits = (int)flat.size(); P.nslots = nslots; P.grid = grid;
    if (P.nunits) {
        if (cudaMalloc(&P.d_units, sizeof(WorkUnit) * flat.size()) != cudaSuccess ||
            cudaMalloc(&P.d_counter, sizeof(int32_t) * (1 + (size_t)std::max(nslots, nhint))) != cudaSuccess ||
            cudaMalloc(&P.d_slotinfo, sizeof(int32_t) * slotinfo.size()) != cudaSuccess)
            return fail(MPCGEMM_ERR_NOMEM, "cudaMalloc plan");
        // uploads ordered on the call's stream (a later call on another stream is ordered after
        // this one by StreamOrder); a pageable-source cudaMemcpyAsync has staged the host data
        // by the time it returns, so the host vectors may go
        CK(cudaMemcpyAsync(P.d_units, flat.data(), sizeof(WorkUnit) * flat.size(), cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(P.d_slotinfo, slotinfo.data(), sizeof(int32_t) * slotinfo.size(), cudaMemcpyHostToDevice, st));
        CK(cudaMemsetAsync(P.d_counter, 0, sizeof(int32_t) * (1 + (size_t)std::max(nslots, nhint)), st));   // counter + k-phase hints
    }
    auto res = g_plans.emplace(std::make_pair(dev, key), P);
    *out = &res.first->second;
    return 0;
}

int sm_count(int dev) {
    int v = 148;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
}

int env_int(const char *name, int dflt) {
    const char *v = getenv(name);
    return v && *v ? atoi(v) : dflt;
}

bool overlaps(const void *a, size_t na, const void *b, size_t nb) {
    const char *x = (const char *)a, *y = (const char *)b;
    return x < y + nb && y < x + na;
}

size_t mat_span(const mpc_rmat &M, int64_t rows, int64_t cols, int L, int which) {
    if (rows == 0 || cols == 0) return 0;
    const size_t ents = (size_t)((rows - 1) * M.ld + cols);
    return which == 0 ? ents : which == 1 ? ents * 8 : ents * 8 * (size_t)L;
}

int check_args(int64_t m, int64_t n, int64_t k, int32_t prec, const mpc_cmat *A, const mpc_cmat *B,
               const mpc_cmat *C, int method, bool check_alias = true) {
    if (!A || !B || !C) return fail(MPCGEMM_ERR_ARG, "null matrix descriptor");
    if (m < 0 || n < 0 || k < 0) return fail(MPCGEMM_ERR_ARG, "negative dimension");
    if (method != MPCGEMM_3M && method != MPCGEMM_4M) return fail(MPCGEMM_ERR_ARG, "method must be 3 or 4");
    if (prec < 2 || prec > 4096) return fail(MPCGEMM_ERR_PREC, "prec outside [2, 4096]");
    if (m > INT32_MAX / 2 || n > INT32_MAX / 2 || k > INT32_MAX / 2) return fail(MPCGEMM_ERR_ARG, "dimension too large");
    const mpc_rmat *mats[6] = {&A->re, &A->im, &B->re, &B->im, &C->re, &C->im};
    const int64_t cols[6] = {k, k, n, n, n, n};
    const int64_t rows[6] = {m, m, k, k, m, m};
    for (int q = 0; q < 6; q++) {
        if (rows[q] == 0 || cols[q] == 0) continue;
        if (!mats[q]->sign || !mats[q]->exp || !mats[q]->limbs) return fail(MPCGEMM_ERR_ARG, "null array");
        if (mats[q]->ld < cols[q]) return fail(MPCGEMM_ERR_ARG, "ld < cols");
    }
    const int L = (prec + 63) / 64;
    if (!check_alias) return 0;
    for (int c = 4; c < 6; c++)
        for (int q = 0; q < 4; q++)
            for (int w = 0; w < 3; w++)
                for (int w2 = 0; w2 < 3; w2++) {
                    const void *pc = w == 0 ? (const void *)mats[c]->sign : w == 1 ? (const void *)mats[c]->exp : (const void *)mats[c]->limbs;
                    const void *pq = w2 == 0 ? (const void *)mats[q]->sign : w2 == 1 ? (const void *)mats[q]->exp : (const void *)mats[q]->limbs;
                    if (overlaps(pc, mat_span(*mats[c], rows[c], cols[c], L, w), pq, mat_span(*mats[q], rows[q], cols[q], L, w2)))
                        return fail(MPCGEMM_ERR_ALIAS, "C overlaps A or B");
                }
    return 0;
}

DMat dm(const mpc_rmat &M) { return DMat{M.sign, M.exp, M.limbs, M.ld}; }
DMatOut dmo(const mpc_rmat &M) { return DMatOut{M.sign, M.exp, M.limbs, M.ld}; }

int64_t nblocks(int64_t m) { return (m + kSBlk - 1) / kSBlk; }

// the small per-call metadata area: eA[m], eB[n], nzA[m], nzB[n], then the flags region:
// validate error flag, the pre-pass results per 256-row block, the per-block slice counts
struct MetaView {
    int64_t *eA, *eB;
    uint8_t *nzA, *nzB;
    uint32_t *errflag;
    unsigned long long *omin, *omin1;
    long long *omax2;
    int32_t *sblk;
    unsigned long long *dmin2, *dmin12;   // device rule: the stage-2 arrays (per block)
    long long *dmax22;
    DevRuleState *drs;                    // device rule: the chosen s / plan
};
size_t meta_flags_off(int64_t m, int64_t n) { return align_up(8 * (m + n) + (m + n) + 64, 256); }
size_t meta_bytes(int64_t m, int64_t n) {
    return meta_flags_off(m, n) + align_up(64 + 52 * (size_t)nblocks(m) + 64, 256) + align_up(sizeof(DevRuleState), 256);
}
MetaView meta_view(uint8_t *meta, int64_t m, int64_t n) {
    MetaView v;
    v.eA = (int64_t *)meta; v.eB = v.eA + m;
    v.nzA = (uint8_t *)(v.eB + n); v.nzB = v.nzA + m;
    uint8_t *flags = meta + meta_flags_off(m, n);
    v.errflag = (uint32_t *)flags;
    v.omin = (unsigned long long *)(flags + 64);
    v.omin1 = v.omin + nblocks(m);
    v.omax2 = (long long *)(v.omin1 + nblocks(m));
    v.sblk = (int32_t *)(v.omax2 + nblocks(m));
    v.dmin2 = (unsigned long long *)align_up((size_t)(v.sblk + nblocks(m)), 8);
    v.dmin12 = v.dmin2 + nblocks(m);
    v.dmax22 = (long long *)(v.dmin12 + nblocks(m));
    v.drs = (DevRuleState *)(meta + meta_flags_off(m, n) + align_up(64 + 52 * (size_t)nblocks(m) + 64, 256));
    return v;
}

// per-block pre-pass integers (minT, minT1, maxD2) of the 256-row blocks of A, and the global
// reduction (the rule's input for one common s)
struct Bounds {
    std::vector<int64_t> minT, minT1, maxD2;
    int64_t g[3] = {-1, -1, -1};
};

// workspace layout of one call
struct Layout {
    size_t meta;      // eA, eB, nz, flags, prepass outputs
    size_t pre;       // pre-pass planes + T partials
    size_t main;      // digit planes + partials
    int64_t kp, nstrips;
};

int tile_bn(int64_t n) { return n > 128 ? 256 : 128; }

// Load-balance target for the MMA k-blocks of one unit: about one unit per CTA (MPCGEMM_BALANCE
// units per CTA; 4 was 21 % slower at config 2: more, shorter units each pay an accumulator drain).  (The
// INT32 exactness cap is separate: exact_cap().)
int64_t chunk_kb(int64_t m, int64_t n, int64_t k, int s, int method, int BM, int BN, int grid) {
    const int64_t KB = (k + kBK - 1) / kBK;
    const int64_t tiles = ((m + BM - 1) / BM) * ((n + BN - 1) / BN) * (BM / 128);   // in 128-row CTA tiles
    const int64_t npairs_total = method == 0 ? 1 : (method == 3 ? 3 : 4);
    const int64_t work = npairs_total * KB * (int64_t)s * (s + 1) / 2 * tiles;   // k-blocks
    int64_t target = work / (std::max(1, env_int("MPCGEMM_BALANCE", 1)) * (int64_t)grid);
    return std::max<int64_t>(8, std::min<int64_t>(target, 1 << 30));
}

// k-blocks one INT32 accumulator may sum; MPCGEMM_MAXKB lowers it
int64_t exact_cap() {
    int e = env_int("MPCGEMM_MAXKB", 0);
    return e > 0 ? std::min<int64_t>(kMaxKBlocksPerChunk, e) : kMaxKBlocksPerChunk;
}

struct Geometry { int BM, BN, grid, maxkb, g2; };

// m_balance (> 0): the row count whose work sets the chunk target -- row groups use the whole
// call's, so every group has the whole call's slot table (and a group's workspace scales with its
// rows)
Geometry main_geometry(int dev, int64_t m, int64_t n, int64_t k, int s, int method, int64_t m_balance = 0) {
    Geometry g;
    g.BN = env_int("MPCGEMM_BN", tile_bn(n));
    if (g.BN != 128 && g.BN != 256) g.BN = tile_bn(n);
    g.BM = (g.BN == 256 && env_int("MPCGEMM_CTA2", 1)) ? 256 : 128;   // CTA pairs for wide tiles
    // MPCGEMM_RESERVE_SMS: SMs left free of the persistent slice GEMM (multi-GPU: NCCL's kernels
    // cannot become resident next to a slice-GEMM CTA -- registers -- so the B broadcast / C gather
    // of neighbouring products overlap the GEMM only on reserved SMs)
    g.grid = std::max(2, sm_count(dev) - std::max(0, env_int("MPCGEMM_RESERVE_SMS", 0)));
    g.maxkb = (int)chunk_kb(m_balance > 0 ? m_balance : m, n, k, s, method, g.BM, g.BN, g.grid);
    // two diagonals per unit (G = 2) halve the operand loads per MMA, but keep a unit's chain of
    // stages as long as one diagonal's; when the G = 2 units are fewer than ~4 per fetching CTA (pair)
    // the call is parallelism-bound and single-diagonal units, which the load-balance target cuts
    // along their (pair, p, k-block) sequence, finish sooner (config 1 46 -> 43 us, config 2 4M
    // 0.388 -> 0.327 ms per call; config 4 / 5's large products keep G = 2).  MPCGEMM_G2 forces it.
    const char *ge = getenv("MPCGEMM_G2");
    if (ge && *ge) g.g2 = atoi(ge) != 0;
    else {
        const int64_t mb = m_balance > 0 ? m_balance : m;
        const int64_t units = ((mb + g.BM - 1) / g.BM) * ((n + g.BN - 1) / g.BN) * ((s + 1) / 2) * 3;
        g.g2 = units >= 4LL * (g.BM == 256 ? g.grid / 2 : g.grid);
    }
    return g;
}

int64_t count_slots(int64_t k, int s, int method, int maxkb, bool g2) {
    Plan P;
    method_jobs(method, P);
    int64_t n = 0;
    for (const Segment &sg : diag_segments(P, (k + kBK - 1) / kBK, s, method, maxkb, g2))
        n += sg.G * sg.nch;
    return n;
}

// g2: the geometry's unit shape (main_geometry().g2) -- it sets the slot count; -1 for s = 0 layouts
Layout layout_for(int64_t m, int64_t n, int64_t k, int s, int method, int maxkb, int prec = 64, bool beta = false,
                  int g2 = -1) {
    Layout Lo;
    Lo.kp = align_up((size_t)std::max<int64_t>(k, 1), 16);
    Lo.nstrips = (std::max<int64_t>(n, 1) + kStrip - 1) / kStrip;
    Lo.meta = meta_bytes(m, n);
    const int64_t KB = (k + kBK - 1) / kBK;
    const int64_t nslotsT = (KB + exact_cap() - 1) / exact_cap();
    Lo.pre = align_up((size_t)(m + n) * Lo.kp, 256) + align_up((size_t)(m + n) * Lo.kp * 4, 256) +
             align_up((size_t)nslotsT * ((m + kRowBlk - 1) / kRowBlk * kRowBlk) * Lo.nstrips * kStrip * 4, 256);
    Lo.main = 0;
    if (s > 0) {
        const int parts = method == 3 ? 3 : 2;
        const int64_t nslots = count_slots(k, s, method, maxkb, g2 < 0 ? g2_enabled() : g2 != 0);
        Lo.main = align_up((size_t)parts * s * m * Lo.kp, 256) + align_up((size_t)parts * s * n * Lo.kp, 256) +
                  align_up((size_t)nslots * ((m + kRowBlk - 1) / kRowBlk * kRowBlk) * Lo.nstrips * kStrip * 4, 256) +
                  align_up(fold_scratch_words(m, (n + kFoldLdAlign - 1) / kFoldLdAlign * kFoldLdAlign, s, (prec + 63) / 64, beta) * 8, 256);
    }
    return Lo;
}

// prepass on device pointers (synchronizes the stream).  Stage 1 gives each block's minT; if
// any block has minT == 0 (or full), stage 2 gives every block's (minT1, maxD2).  Blocks
// without a nonzero line pair keep -1.  B->g is the reduction over blocks (the global pre-pass).
int run_prepass(int dev, int64_t m, int64_t n, int64_t k, int32_t prec, const mpc_cmat *A, const mpc_cmat *B,
                int full, cudaStream_t st, uint8_t *meta, uint8_t *pre, const Layout &Lo, int simt, Bounds *out,
                const uint8_t *tb = nullptr) {
    const int L = (prec + 63) / 64;
    const MetaView mv = meta_view(meta, m, n);
    const int64_t nb = nblocks(m);
    int8_t *tA = (int8_t *)pre, *tB = tA + m * Lo.kp;
    int32_t *relA = (int32_t *)(pre + align_up((size_t)(m + n) * Lo.kp, 256)), *relB = relA + m * Lo.kp;
    int32_t *T = (int32_t *)(pre + align_up((size_t)(m + n) * Lo.kp, 256) + align_up((size_t)(m + n) * Lo.kp * 4, 256));
    CK(prepass_planes2_launch(dm(A->re), dm(A->im), dm(B->re), dm(B->im), m, n, k, Lo.kp, L, mv.eA, mv.eB, tA, relA, tB,
                              relB, st, nullptr, 0, nullptr, 0, tb));
    const int BN = tile_bn(n);
    const int grid = sm_count(dev);
    PlanKey key{m, n, k, 1, 0, 128, BN, grid, simt, (int)kMaxKBlocksPerChunk, 0, 0, {}};
    Plan *plan;
    if (int rc = build_plan(dev, key, &plan, st)) return rc;
    SliceGemmLaunch SL;
    memset(&SL, 0, sizeof(SL));
    SL.P.units = plan->d_units; SL.P.nunits = plan->nunits; SL.P.counter = plan->d_counter;
    SL.P.partials = T; SL.P.nslots = plan->nslots; SL.P.nstrips = Lo.nstrips;
    SL.P.m = (int32_t)m; SL.P.n = (int32_t)n; SL.P.s = 1; SL.P.KB = (int32_t)((k + kBK - 1) / kBK);
    SL.P.kk_last = (int32_t)(((k - 1) % kBK) / 32 + 1) % (kBK / 32);
    SL.P.partsA = SL.P.partsB = 1;
    for (int q = 0; q < kMaxJobs; q++) SL.P.jobs[q] = plan->jobs[q];
    SL.digA = tA; SL.digB = tB; SL.rowsA = m; SL.rowsB = n; SL.kp = Lo.kp;
    SL.grid = plan->grid; SL.BM = 128; SL.BN = BN; SL.simt = simt; SL.nunits = plan->nunits; SL.units_flat = plan->d_units;
    CK(slicegemm_launch(SL, st));
    std::vector<unsigned long long> h(3 * nb);
    // minima start at ~0, the max-plus maximum at -1: all bytes 0xFF (no pageable host copy)
    CK(cudaMemsetAsync(mv.omin, 0xFF, 8 * 3 * nb, st));
    CK(prepass_reduce_launch(T, plan->nslots, Lo.nstrips, m, n, k, Lo.kp, mv.nzA, mv.nzB, relA, relB, 1,
                             mv.omin, mv.omin1, mv.omax2, st));
    if (int rc = readback(dev, h.data(), mv.omin, 8 * nb, st)) return rc;
    out->minT.assign(nb, -1); out->minT1.assign(nb, -1); out->maxD2.assign(nb, -1);
    bool any0 = false;
    for (int64_t b = 0; b < nb; b++) {
        out->minT[b] = h[b] == ~0ull ? -1 : (int64_t)h[b];
        out->minT1[b] = out->minT[b];
        any0 = any0 || out->minT[b] == 0;
    }
    if (any0 || full) {
        CK(cudaMemsetAsync(mv.omin, 0xFF, 8 * 3 * nb, st));
        CK(prepass_reduce_launch(T, plan->nslots, Lo.nstrips, m, n, k, Lo.kp, mv.nzA, mv.nzB, relA, relB, 2,
                                 mv.omin, mv.omin1, mv.omax2, st));
        if (int rc = readback(dev, h.data(), mv.omin, 8 * 3 * nb, st)) return rc;
        for (int64_t b = 0; b < nb; b++) {
            out->minT[b] = h[b] == ~0ull ? -1 : (int64_t)h[b];
            out->minT1[b] = h[nb + b] == ~0ull ? -1 : (int64_t)h[nb + b];
            out->maxD2[b] = (int64_t)h[2 * nb + b];
        }
    }
    // global: MIN minT; if it is 0 (or full) MIN minT1 and MAX maxD2, else (minT, minT, -1)
    int64_t g0 = -1, g1 = -1, g2 = -1;
    for (int64_t b = 0; b < nb; b++) {
        if (out->minT[b] >= 0 && (g0 < 0 || out->minT[b] < g0)) g0 = out->minT[b];
        if (out->minT1[b] >= 0 && (g1 < 0 || out->minT1[b] < g1)) g1 = out->minT1[b];
        if (out->maxD2[b] > g2) g2 = out->maxD2[b];
    }
    if (g0 < 0) { out->g[0] = out->g[1] = out->g[2] = -1; }
    else if (g0 > 0 && !full) { out->g[0] = g0; out->g[1] = g0; out->g[2] = -1; }
    else { out->g[0] = g0; out->g[1] = g1; out->g[2] = g2; }
    return 0;
}

// b = 53 - ceil((53 + ceil(log2 k)) / 2): the paper's binary64 slice width
int fp64_slice_bits(int64_t k) {
    int lk = 0;
    while ((1ll << lk) < k) lk++;
    return 53 - (53 + lk + 1) / 2;
}

struct F64Plan {
    int4 *d_units = nullptr;
    JobDesc *d_jobs = nullptr;
    int nunits = 0;
};
std::map<std::tuple<int, int64_t, int64_t, int, int>, F64Plan> g_f64plans;

// NEXT-1 path: binary64 digits on FP64 DMMA (fp64path.cu)
int run_main_f64(int dev, int64_t m, int64_t n, int64_t k, int32_t prec, const mpc_cmat *A, const mpc_cmat *B,
                 mpc_cmat *C, int method, int s, int b, cudaStream_t st, uint8_t *meta, uint8_t *big,
                 mpcgemm_report *rep, StageEvents *E) {
    const int L = (prec + 63) / 64;
    int64_t *eA = (int64_t *)meta, *eB = eA + m;
    const int parts = method == 3 ? 3 : 2;
    const int64_t kp = (int64_t)align_up((size_t)k, 16);
    double *digA = (double *)big;
    double *digB = (double *)((uint8_t *)digA + align_up((size_t)parts * s * m * kp * 8, 256));
    int64_t *partials = (int64_t *)((uint8_t *)digB + align_up((size_t)parts * s * n * kp * 8, 256));
    CK(split_f64_launch(dm(A->re), dm(A->im), 0, m, k, kp, L, eA, s, b, parts, digA, st));
    CK(split_f64_launch(dm(B->re), dm(B->im), 1, n, k, kp, L, eB, s, b, parts, digB, st));
    if (E) CK(cudaEventRecord(E->ev[3], st));
    auto key = std::make_tuple(dev, m, n, s, method);
    auto it = g_f64plans.find(key);
    if (it == g_f64plans.end()) {
        Plan P;
        method_jobs(method, P);
        std::vector<int4> units;
        const int tm = (int)((m + 63) / 64), tn = (int)((n + 63) / 64);
        for (int r = s + 1; r >= 2; r--)                   // longest diagonals first
            for (int q = 0; q < P.njobs; q++)
                for (int a = 0; a < tm; a++)
                    for (int c = 0; c < tn; c++) units.push_back(make_int4(q, a, c, r));
        F64Plan F;
        F.nunits = (int)units.size();
        if (cudaMalloc(&F.d_units, sizeof(int4) * units.size()) != cudaSuccess ||
            cudaMalloc(&F.d_jobs, sizeof(JobDesc) * kMaxJobs) != cudaSuccess)
            return fail(MPCGEMM_ERR_NOMEM, "cudaMalloc f64 plan");
        CK(cudaMemcpyAsync(F.d_units, units.data(), sizeof(int4) * units.size(), cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(F.d_jobs, P.jobs, sizeof(JobDesc) * kMaxJobs, cudaMemcpyHostToDevice, st));
        it = g_f64plans.emplace(key, F).first;
    }
    CK(dmma_slicegemm_launch(digA, digB, m, n, kp, s, it->second.d_units, it->second.nunits, it->second.d_jobs,
                             3, partials, st));
    if (E) CK(cudaEventRecord(E->ev[4], st));
    CK(fold_f64_launch(partials, m, n, s, b, method, prec, L, eA, eB, dmo(C->re), dmo(C->im), st));
    if (E) CK(cudaEventRecord(E->ev[5], st));
    if (rep) {
        rep->kernel_launches += 4;
        rep->work_units = it->second.nunits;
        rep->slicegemm_ctas = it->second.nunits;
        rep->mma_instructions = 0;
    }
    return 0;
}

size_t f64_main_bytes(int64_t m, int64_t n, int64_t k, int s, int method) {
    const int parts = method == 3 ? 3 : 2;
    const int64_t kp = (int64_t)align_up((size_t)std::max<int64_t>(k, 1), 16);
    return align_up((size_t)parts * s * m * kp * 8, 256) + align_up((size_t)parts * s * n * kp * 8, 256) +
           align_up((size_t)3 * (s + 2) * m * n * 8, 256);
}

mpc_cmat rows_of(const mpc_cmat &M, int64_t r0, int L) {
    mpc_cmat v = M;
    for (mpc_rmat *R : {&v.re, &v.im}) {
        const int64_t o = r0 * R->ld;
        R->sign += o; R->exp += o; R->limbs += o * L;
    }
    return v;
}

// row groups of the e2e path: the hook runs after group [r0, r1) of C is final (stream order)
using GroupHook = std::function<int(int64_t, int64_t)>;

// the device hot path with a known workspace.  group_rows > 0 (a multiple of 256): the rows of
// A / C are processed in groups of that many rows (split A_g, slice GEMM, fold), B split once;
// Lo must then be the layout of one group.
int run_main(int dev, int64_t m, int64_t n, int64_t k, int32_t prec, const mpc_cmat *A, const mpc_cmat *B,
             mpc_cmat *C, int method, int s, cudaStream_t st, uint8_t *meta, uint8_t *big, const Layout &Lo,
             int simt, mpcgemm_report *rep, StageEvents *E, int beta, int alpha_neg,
             const std::vector<int32_t> &sblk, int64_t group_rows = 0, const GroupHook *hook = nullptr,
             unsigned long long *mma_dev = nullptr) {
    const int L = (prec + 63) / 64;
    const MetaView mv = meta_view(meta, m, n);
    int64_t *eA = mv.eA, *eB = mv.eB;
    const int parts = method == 3 ? 3 : 2;
    const int64_t mg = group_rows > 0 ? std::min(m, group_rows) : m;
    int8_t *digA = (int8_t *)big;
    int8_t *digB = digA + align_up((size_t)parts * s * mg * Lo.kp, 256);
    int32_t *partials = (int32_t *)((uint8_t *)digB + align_up((size_t)parts * s * n * Lo.kp, 256));
    uint64_t *fix = (uint64_t *)((uint8_t *)partials);  // set below per plan
    const bool one_group = mg >= m;                   // B and A split by one launch
    int nsplit = 1;
    {
        Nvtx r(one_group ? "mpcgemm.a3_split" : "mpcgemm.a3_split_B");
        if (one_group) CK(split2_launch(dm(A->re), dm(A->im), dm(B->re), dm(B->im), m, n, k, Lo.kp, L, eA, eB, s, parts,
                                        digA, digB, st, nullptr, &nsplit));
        else CK(split_launch(dm(B->re), dm(B->im), 1, n, k, Lo.kp, L, eB, s, parts, digB, st));
    }
    if (!sblk.empty()) CK(cudaMemcpyAsync(mv.sblk, sblk.data(), 4 * sblk.size(), cudaMemcpyHostToDevice, st));
    int launches = one_group ? nsplit - 1 : 1;         // (+ 3 per group below: split A, GEMM, fold)
    for (int64_t r0 = 0; r0 < m; r0 += mg) {
        const int64_t mr = std::min(mg, m - r0);
        const mpc_cmat Ag = rows_of(*A, r0, L);
        const mpc_cmat Cg = rows_of(*C, r0, L);
        if (!one_group) {
            Nvtx r("mpcgemm.a3_split_A");
            CK(split_launch(dm(Ag.re), dm(Ag.im), 0, mr, k, Lo.kp, L, eA + r0, s, parts, digA, st));
        }
        if (E && r0 == 0) CK(cudaEventRecord(E->ev[3], st));
        const Geometry geo = main_geometry(dev, mr, n, k, s, method, m);
        const int BN = geo.BN;
        std::vector<int32_t> sb;
        if (!sblk.empty()) sb.assign(sblk.begin() + (r0 >> kSBlkShift), sblk.begin() + ((r0 + mr + kSBlk - 1) >> kSBlkShift));
        PlanKey key{mr, n, k, s, method, geo.BM, BN, geo.grid, simt, geo.maxkb, geo.g2,
                    env_int("MPCGEMM_ORDER", 2), sb};
        Plan *plan;
        if (int rc = build_plan(dev, key, &plan, st)) return rc;
        SliceGemmLaunch SL;
        memset(&SL, 0, sizeof(SL));
        SL.P.units = plan->d_units; SL.P.nunits = plan->nunits; SL.P.counter = plan->d_counter;
        SL.P.partials = partials; SL.P.nslots = plan->nslots; SL.P.nstrips = Lo.nstrips;
        SL.P.m = (int32_t)mr; SL.P.n = (int32_t)n; SL.P.s = s; SL.P.KB = (int32_t)((k + kBK - 1) / kBK);
        SL.P.kk_last = (int32_t)(((k - 1) % kBK) / 32 + 1) % (kBK / 32);
        SL.P.partsA = SL.P.partsB = parts;
        SL.P.dbg = env_int("MPCGEMM_DBG", 0);
        SL.P.hot = env_int("MPCGEMM_KPHASE", 2) ? plan->d_counter + 1 : nullptr;
        SL.P.pblk = env_int("MPCGEMM_PBLK", 64);
        SL.P.kmode = kphase_mode(SL.P.KB);
        SL.P.mma_count = mma_dev;
        SL.P.halfn = env_int("MPCGEMM_HALFN", 1);
        for (int q = 0; q < kMaxJobs; q++) SL.P.jobs[q] = plan->jobs[q];
        SL.digA = digA; SL.digB = digB; SL.rowsA = mr; SL.rowsB = n; SL.kp = Lo.kp;
        SL.grid = plan->grid; SL.BM = geo.BM; SL.BN = BN; SL.simt = simt; SL.nunits = plan->nunits;
        SL.units_flat = plan->d_units;
        if (!(SL.P.dbg & 16)) {                        // (MPCGEMM_DBG bit 4: fold the previous call's
            Nvtx r("mpcgemm.a4_slicegemm");            //  partials again -- a race detector for the fold)
            CK(slicegemm_launch(SL, st));
        }
        if (E && r0 + mr >= m) CK(cudaEventRecord(E->ev[4], st));
        FoldParams F{};
        F.partials = partials; F.nslots = plan->nslots; F.nstrips = Lo.nstrips; F.m = mr; F.n = n;
        F.s = s; F.method = method; F.prec = prec; F.L = L; F.slotinfo = plan->d_slotinfo;
        F.eA = eA + r0; F.eB = eB; F.Cre = dmo(Cg.re); F.Cim = dmo(Cg.im);
        F.beta = beta; F.alpha_neg = alpha_neg; F.C0re = dm(Cg.re); F.C0im = dm(Cg.im);
        F.ldF = (n + kFoldLdAlign - 1) / kFoldLdAlign * kFoldLdAlign;
        F.sblk = sblk.empty() ? nullptr : mv.sblk + (r0 >> kSBlkShift);    // NEXT-4: per-block triangles
        F.uni1 = plan->uni1 ? 1 : 0;
        F.unic = plan->unic ? 1 : 0;
        F.norm_generic = env_int("MPCGEMM_NORM_GENERIC", 0);
        F.l2hint = env_int("MPCGEMM_FOLD_L2HINT", 1);
        fix = (uint64_t *)((uint8_t *)partials +
                           align_up((size_t)plan->nslots * ((mr + kRowBlk - 1) / kRowBlk * kRowBlk) * Lo.nstrips * kStrip * 4, 256));
        F.fix = fix;
        {
            Nvtx r("mpcgemm.a5a6_fold_normalize");
            CK(fold_normalize_launch(F, st));
        }
        launches += 3;                                 // split A_g, slice GEMM, fold
        if (rep) {
            rep->mma_instructions += plan->mma; rep->work_units += plan->nunits;
            rep->partial_slots = (int32_t)plan->nslots;
            rep->slicegemm_ctas = simt ? plan->nunits : plan->grid;
            rep->tile_m = geo.BM; rep->tile_n = BN;
        }
        if (hook) if (int rc = (*hook)(r0, r0 + mr)) return rc;
    }
    if (E) CK(cudaEventRecord(E->ev[5], st));
    if (rep) rep->kernel_launches += launches;
    return 0;
}

// ---------------------------------------------------------------- device-rule mode
// Candidate plans for every s the device rule can pick without needing more than planned: the
// rule's s at log2 rho-hat = 0 (the smallest) .. at minT = 1 (the largest first-stage s).
struct DevPlanSet {
    DevPlan *d_plans = nullptr;          // [s_hi - s_lo + 1]
    int32_t *d_counter = nullptr;        // the shared unit counter
    int s_lo = 0, s_hi = 0;
    int64_t nslots_max = 0;
    bool uni1 = true;                    // every candidate has one chunk per (job, diagonal)
    bool unic = true;                    // every candidate: equal chunk counts across the jobs
    bool chunked_unic = false;           // some candidate has (chunk, job) slot order with > 1 chunk
    size_t main_bytes = 0;               // workspace of the largest candidate
};
std::map<std::tuple<int, int64_t, int64_t, int64_t, int, int, int, int>, DevPlanSet> g_devplans;

int dev_plan_set(int dev, int64_t m, int64_t n, int64_t k, int32_t prec, int method, cudaStream_t st,
                 DevPlanSet **out) {
    const int s_lo = rule_slices(prec, method, 0.0);
    const int s_hi = rule_slices(prec, method, rule_log2rho(k, 1, 1, -1));
    if (s_lo < 0 || s_hi < 0) return fail(MPCGEMM_ERR_SLICES, "device rule: slice range above 1024");
    auto key = std::make_tuple(dev, m, n, k, method, s_lo, s_hi, env_int("MPCGEMM_ORDER", 2));
    auto it = g_devplans.find(key);
    if (it != g_devplans.end()) { *out = &it->second; return 0; }
    DevPlanSet S;
    S.s_lo = s_lo; S.s_hi = s_hi;
    std::vector<DevPlan> hp;
    // one unit shape (G = 2 or single diagonals) for every candidate, so their slot orders agree
    const int g2c = main_geometry(dev, m, n, k, s_hi, method).g2;
    for (int s = s_lo; s <= s_hi; s++) {
        Geometry geo = main_geometry(dev, m, n, k, s, method);
        geo.g2 = g2c;
        PlanKey key2{m, n, k, s, method, geo.BM, geo.BN, geo.grid, 0, geo.maxkb, geo.g2,
                     env_int("MPCGEMM_ORDER", 2), {}};
        Plan *plan;
        if (int rc = build_plan(dev, key2, &plan, st)) return rc;
        hp.push_back(DevPlan{plan->d_units, plan->d_counter + 1, plan->d_slotinfo, s, plan->nunits, plan->nslots, 0});
        S.nslots_max = std::max<int64_t>(S.nslots_max, plan->nslots);
        S.uni1 = S.uni1 && plan->uni1;
        S.unic = S.unic && plan->unic;
        S.chunked_unic = S.chunked_unic || (plan->unic && !plan->uni1);
        S.main_bytes = std::max(S.main_bytes, layout_for(m, n, k, s, method, geo.maxkb, prec, false, geo.g2).main);
    }
    // one fold variant serves every candidate: their slot orders must agree (with the present job
    // structures a chunked (chunk, job)-ordered plan is 3M, and then every candidate is)
    if (!S.unic && S.chunked_unic) return fail(MPCGEMM_ERR_ARG, "device rule: candidate plans with different slot orders");
    if (cudaMalloc(&S.d_plans, sizeof(DevPlan) * hp.size()) != cudaSuccess ||
        cudaMalloc(&S.d_counter, sizeof(int32_t)) != cudaSuccess)
        return fail(MPCGEMM_ERR_NOMEM, "cudaMalloc device plans");
    CK(cudaMemcpyAsync(S.d_plans, hp.data(), sizeof(DevPlan) * hp.size(), cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(S.d_counter, 0, sizeof(int32_t), st));   // then re-armed by each launch's last fetch
    *out = &g_devplans.emplace(key, S).first->second;
    return 0;
}

// the device-rule hot path: pre-pass, stage 2 (device-gated), rule kernel, then split / slice GEMM
// / fold reading the chosen plan from device memory -- no host synchronisation anywhere
int run_device_rule(int dev, int64_t m, int64_t n, int64_t k, int32_t prec, const mpc_cmat *A, const mpc_cmat *B,
                    mpc_cmat *C, int method, cudaStream_t st, uint8_t *meta, DevCache &dc, const mpcgemm_opts *opts,
                    mpcgemm_report *rep) {
    const int L = (prec + 63) / 64;
    const MetaView mv = meta_view(meta, m, n);
    DevPlanSet *S;
    if (int rc = dev_plan_set(dev, m, n, k, prec, method, st, &S)) return rc;
    const int s_hi = S->s_hi;
    const Layout Lo = layout_for(m, n, k, 0, method, kMaxKBlocksPerChunk);
    // workspace: pre-pass area and the largest candidate's main area share the cache (pre-pass first)
    const size_t need = std::max(Lo.pre, S->main_bytes);
    uint8_t *big;
    if (opts && opts->workspace) {
        if (opts->workspace_bytes < need) return fail(MPCGEMM_ERR_NOMEM, "caller workspace too small");
        big = (uint8_t *)opts->workspace;
    } else {
        if (int rc = grow(&dc.ws, &dc.ws_bytes, need)) return rc;
        big = (uint8_t *)dc.ws;
    }
    // ---- a-2 pre-pass on the device (as run_prepass, without the readback)
    int8_t *tA = (int8_t *)big, *tB = tA + m * Lo.kp;
    int32_t *relA = (int32_t *)(big + align_up((size_t)(m + n) * Lo.kp, 256)), *relB = relA + m * Lo.kp;
    int32_t *T = (int32_t *)(big + align_up((size_t)(m + n) * Lo.kp, 256) + align_up((size_t)(m + n) * Lo.kp * 4, 256));
    {
        Nvtx r("mpcgemm.a2_prepass_device_rule");
        const int64_t nb = nblocks(m);
        const bool small_pre = prepass_small(m, n, k);
        // (the planes kernel also sets the stage-1 minima and the max-plus/rule targets -- with the
        //  rule's done counter after them -- to all ones)
        CK(prepass_planes2_launch(dm(A->re), dm(A->im), dm(B->re), dm(B->im), m, n, k, Lo.kp, L, mv.eA, mv.eB, tA, relA,
                                  tB, relB, st, mv.omin, 3 * nb, mv.dmin2, 3 * nb + 1,
                                  planes_tb_on() ? (uint8_t *)dc.tb : nullptr));
        if (small_pre) {                               // T (dp4a) + stage 1 in one launch, T as one plane
            CK(prepass_small_t_launch(tA, tB, m, n, k, Lo.kp, mv.nzA, mv.nzB, T, Lo.nstrips, mv.omin, st));
            CK(prepass_rule_launch(T, 1, Lo.nstrips, m, n, k, Lo.kp, mv.nzA, mv.nzB, relA, relB, mv.omin, mv.dmin2,
                                   mv.dmin12, mv.dmax22, prec, method, S->d_plans, S->s_lo, s_hi, mv.drs, st));
        } else {
            PlanKey key{m, n, k, 1, 0, 128, tile_bn(n), sm_count(dev), 0, (int)kMaxKBlocksPerChunk, 0, 0, {}};
            Plan *plan;
            if (int rc = build_plan(dev, key, &plan, st)) return rc;
            SliceGemmLaunch SL;
            memset(&SL, 0, sizeof(SL));
            SL.P.units = plan->d_units; SL.P.nunits = plan->nunits; SL.P.counter = plan->d_counter;
            SL.P.partials = T; SL.P.nslots = plan->nslots; SL.P.nstrips = Lo.nstrips;
            SL.P.m = (int32_t)m; SL.P.n = (int32_t)n; SL.P.s = 1; SL.P.KB = (int32_t)((k + kBK - 1) / kBK);
            SL.P.kk_last = (int32_t)(((k - 1) % kBK) / 32 + 1) % (kBK / 32);
            SL.P.partsA = SL.P.partsB = 1;
            for (int q = 0; q < kMaxJobs; q++) SL.P.jobs[q] = plan->jobs[q];
            SL.digA = tA; SL.digB = tB; SL.rowsA = m; SL.rowsB = n; SL.kp = Lo.kp;
            SL.grid = plan->grid; SL.BM = 128; SL.BN = tile_bn(n); SL.simt = 0; SL.nunits = plan->nunits;
            SL.units_flat = plan->d_units;
            CK(slicegemm_launch(SL, st));
            CK(prepass_reduce_launch(T, plan->nslots, Lo.nstrips, m, n, k, Lo.kp, mv.nzA, mv.nzB, relA, relB, 1,
                                     mv.omin, mv.omin1, mv.omax2, st));
            CK(prepass_rule_launch(T, plan->nslots, Lo.nstrips, m, n, k, Lo.kp, mv.nzA, mv.nzB, relA, relB, mv.omin,
                                   mv.dmin2, mv.dmin12, mv.dmax22, prec, method, S->d_plans, S->s_lo, s_hi, mv.drs, st));
        }
    }
    // ---- a-3..a-6 with the chosen plan (the workspace laid out for the largest candidate)
    const int parts = method == 3 ? 3 : 2;
    int8_t *digA = (int8_t *)big;
    int8_t *digB = digA + align_up((size_t)parts * s_hi * m * Lo.kp, 256);
    int32_t *partials = (int32_t *)((uint8_t *)digB + align_up((size_t)parts * s_hi * n * Lo.kp, 256));
    uint64_t *fix = (uint64_t *)((uint8_t *)partials +
                                 align_up((size_t)S->nslots_max * ((m + kRowBlk - 1) / kRowBlk * kRowBlk) * Lo.nstrips * kStrip * 4, 256));
    int nsplit = 1;
    {
        Nvtx r("mpcgemm.a3_split");
        CK(split2_launch(dm(A->re), dm(A->im), dm(B->re), dm(B->im), m, n, k, Lo.kp, L, mv.eA, mv.eB, s_hi, parts, digA,
                         digB, st, mv.drs, &nsplit));
    }
    const Geometry geo = main_geometry(dev, m, n, k, s_hi, method);
    SliceGemmLaunch SL;
    memset(&SL, 0, sizeof(SL));
    Plan Pj;
    method_jobs(method, Pj);
    SL.P.counter = S->d_counter; SL.P.partials = partials; SL.P.nstrips = Lo.nstrips;
    SL.P.m = (int32_t)m; SL.P.n = (int32_t)n; SL.P.s = s_hi; SL.P.KB = (int32_t)((k + kBK - 1) / kBK);
    SL.P.kk_last = (int32_t)(((k - 1) % kBK) / 32 + 1) % (kBK / 32);
    SL.P.partsA = SL.P.partsB = parts;
    SL.P.pblk = env_int("MPCGEMM_PBLK", 64);
    SL.P.kmode = kphase_mode(SL.P.KB);
    SL.P.drs = mv.drs;
    SL.P.halfn = env_int("MPCGEMM_HALFN", 1);
    for (int q = 0; q < kMaxJobs; q++) SL.P.jobs[q] = Pj.jobs[q];
    SL.digA = digA; SL.digB = digB; SL.rowsA = m; SL.rowsB = n; SL.kp = Lo.kp;
    SL.grid = geo.BM == 256 ? (geo.grid & ~1) : geo.grid; SL.BM = geo.BM; SL.BN = geo.BN; SL.simt = 0;
    {
        Nvtx r("mpcgemm.a4_slicegemm");
        CK(slicegemm_launch(SL, st));
    }
    FoldParams F{};
    F.partials = partials; F.nstrips = Lo.nstrips; F.m = m; F.n = n;
    F.s = s_hi; F.method = method; F.prec = prec; F.L = L;
    F.eA = mv.eA; F.eB = mv.eB; F.Cre = dmo(C->re); F.Cim = dmo(C->im);
    F.beta = 0; F.alpha_neg = 0; F.C0re = dm(C->re); F.C0im = dm(C->im);
    F.ldF = (n + kFoldLdAlign - 1) / kFoldLdAlign * kFoldLdAlign;
    F.fix = fix; F.drs = mv.drs; F.nslots = S->nslots_max; F.uni1 = S->uni1 ? 1 : 0; F.unic = S->unic ? 1 : 0;
    F.norm_generic = env_int("MPCGEMM_NORM_GENERIC", 0);
    F.l2hint = env_int("MPCGEMM_FOLD_L2HINT", 1);
    {
        Nvtx r("mpcgemm.a5a6_fold_normalize");
        CK(fold_normalize_launch(F, st));
    }
    if (rep) {
        rep->slices = 0;                                 // chosen on the device: mpcgemm_device_rule_result()
        // planes, T GEMM, min, max-plus + rule (one launch unless MPCGEMM_RULE_SEPARATE), split, GEMM, fold;
        // small shapes: planes, T by dp4a + stage 1, max-plus + rule, split, GEMM, fold
        rep->kernel_launches += (prepass_small(m, n, k) ? 4 : 5) + (getenv("MPCGEMM_RULE_SEPARATE") ? 2 : 1) + nsplit;
        rep->slicegemm_ctas = SL.grid; rep->tile_m = geo.BM; rep->tile_n = geo.BN;
        rep->certified = 1;
    }
    return 0;
}

// check_alias = false: the LU's in-place trailing update, whose A22 / L21 / U12 views of one
// matrix interleave in memory but are element-disjoint (the split reads L21, U12 before the
// fold writes A22, in stream order)
// group_rows / hook: the e2e path's row groups (run_main)
int gemm_impl(int64_t m, int64_t n, int64_t k, int32_t prec, const mpc_cmat *A, const mpc_cmat *B, mpc_cmat *C,
              int method, const mpcgemm_opts *opts, mpcgemm_report *rep, bool check_alias = true,
              int64_t group_rows = 0, const GroupHook *hook = nullptr) {
    if (int rc = check_args(m, n, k, prec, A, B, C, method, check_alias)) return rc;
    cudaStream_t st = opts ? (cudaStream_t)opts->stream : nullptr;
    const int forced = opts ? opts->slices : 0;
    const int validate = opts ? opts->validate : 0;
    const int beta = opts ? (opts->beta != 0) : 0;
    const int alpha_neg = opts ? (opts->alpha_neg != 0) : 0;
    const int carrier = opts ? opts->carrier : 0;
    const int adaptive = opts ? (opts->adaptive != 0) : 0;
    const int simt = env_int("MPCGEMM_SLICEGEMM_SIMT", 0);
    if (adaptive && carrier == 1) return fail(MPCGEMM_ERR_ARG, "adaptive slices need the INT8 carrier");
    if (carrier != 0 && carrier != 1) return fail(MPCGEMM_ERR_ARG, "carrier must be 0 (INT8) or 1 (FP64)");
    if (carrier == 1 && (beta || alpha_neg)) return fail(MPCGEMM_ERR_ARG, "beta / alpha_neg need the INT8 carrier");
    const int bits = carrier == 1 ? fp64_slice_bits(k) : 8;
    if (forced < 0 || forced > kMaxSlices) return fail(MPCGEMM_ERR_SLICES, "forced slices outside [1, 1024]");
    if (rep) { memset(rep, 0, sizeof(*rep)); rep->minT = rep->minT1 = rep->maxD2 = -1; rep->mma_issued = -1; }
    const int L = (prec + 63) / 64;
    if (m == 0 || n == 0) return 0;
    if (k == 0) {                                      // A B = 0: C := beta C
        if (!beta) { CK(zero_output_launch(dmo(C->re), m, n, L, st)); CK(zero_output_launch(dmo(C->im), m, n, L, st)); }
        return 0;
    }
    int dev = 0;
    CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(g_mu);
    DevCache &dc = g_cache[dev];
    StreamOrder order(dc, st);
    StageEvents *E = (opts && opts->timing) ? stage_events(dev) : nullptr;
    if (E) CK(cudaEventRecord(E->ev[0], st));
    Layout Lo = layout_for(m, n, k, 0, method, kMaxKBlocksPerChunk);
    if (int rc = grow(&dc.meta, &dc.meta_bytes, Lo.meta)) return rc;
    uint8_t *meta = (uint8_t *)dc.meta;
    const MetaView mv = meta_view(meta, m, n);
    int64_t *eA = mv.eA;                               // (eB = eA + m, nzB = nzA + m: one a-1 launch for both)
    uint8_t *nzA = mv.nzA;
    uint32_t *errflag = mv.errflag;
    Nvtx range_call("mpcgemm");
    if (validate) CK(cudaMemsetAsync(errflag, 0, 4, st));
    int lm_launches = 0;
    const bool devrule = opts && opts->device_rule && !forced && !adaptive && carrier == 0 && !simt && !validate &&
                         !beta && !alpha_neg && group_rows == 0 && !hook;
    // device-rule calls (no host synchronisation inside): programmatic dependent launches
    struct PdlScope {
        int prev;
        explicit PdlScope(bool on) : prev(g_pdl) { g_pdl = on && env_int("MPCGEMM_PDL", 1) != 0; }
        ~PdlScope() { g_pdl = prev; }
    } pdl_scope(devrule);
    {
        Nvtx r("mpcgemm.a1_linemax");
        const size_t lm_need = 8 * (size_t)(m + n) + 16;
        if (planes_tb_on()) {
            if (int rc = grow(&dc.tb, &dc.tb_bytes, 2 * (size_t)(m + n) * Lo.kp)) return rc;
        }
        if (dc.lm_bytes < lm_need) {
            if (int rc = grow(&dc.lm, &dc.lm_bytes, lm_need)) return rc;
            CK(cudaMemsetAsync(dc.lm, 0, dc.lm_bytes, st));
        }
        CK(linemax2_launch(dm(A->re), dm(A->im), dm(B->re), dm(B->im), m, n, k, L, prec, eA, nzA, errflag, validate, st,
                           &lm_launches, (unsigned long long *)dc.lm,
                           planes_tb_on() ? (uint8_t *)dc.tb : nullptr, Lo.kp));
    }
    if (E) CK(cudaEventRecord(E->ev[1], st));
    int launches = lm_launches + (validate ? 1 : 0);   // linemax (A and B, decode fused) [, flag readback]
    if (validate) {
        uint32_t h = 0;
        if (int rc = readback(dev, &h, errflag, 4, st)) return rc;
        if (h & 2u) return fail(MPCGEMM_ERR_EXP_RANGE, "|exp| > 2^61");
        if (h & 1u) return fail(MPCGEMM_ERR_NOT_NORMALIZED, "mantissa not normalized");
    }
    if (devrule) {
        if (rep) rep->kernel_launches = launches;
        return run_device_rule(dev, m, n, k, prec, A, B, C, method, st, meta, dc, opts, rep);
    }
    int s = forced;
    int64_t pb[3] = {-1, -1, -1};
    double log2rho = 0.0;
    std::vector<int32_t> sblk;                         // NEXT-4 per-block slice counts
    if (!s) {
        if (int rc = grow(&dc.ws, &dc.ws_bytes, Lo.pre)) return rc;
        Bounds bd;
        Nvtx range_pre("mpcgemm.a2_prepass");
        if (int rc = run_prepass(dev, m, n, k, prec, A, B, 0, st, meta, (uint8_t *)dc.ws, Lo, simt, &bd,
                                 planes_tb_on() ? (uint8_t *)dc.tb : nullptr))
            return rc;
        for (int q = 0; q < 3; q++) pb[q] = bd.g[q];
        launches += 4 + (pb[0] == 0 ? 2 : 0);         // planes, T GEMM, min, readback [, max-plus, readback]
        log2rho = rule_log2rho(k, pb[0], pb[1], pb[2]);
        s = rule_slices(prec, method, log2rho, bits);
        if (s < 0) return fail(MPCGEMM_ERR_SLICES, "slice rule needs s > 1024");
        if (adaptive) {
            // each 256-row block's own certified s (its rows against all of B); s = the max
            int smin = s;
            sblk.resize(bd.minT.size());
            for (size_t b = 0; b < sblk.size(); b++) {
                const int sb = rule_slices(prec, method, rule_log2rho(k, bd.minT[b], bd.minT1[b], bd.maxD2[b]), 8);
                if (sb < 0) return fail(MPCGEMM_ERR_SLICES, "slice rule needs s > 1024");
                sblk[b] = sb;
                smin = std::min(smin, sb);
            }
            if (smin == s) sblk.clear();               // uniform: the plain path, bit-identical
        }
    }
    if (opts && opts->block_slices) {
        for (int64_t b = 0; b < nblocks(m); b++) opts->block_slices[b] = sblk.empty() ? s : sblk[(size_t)b];
    }
    if (carrier == 1) {
        uint8_t *big;
        if (int rc = grow(&dc.ws, &dc.ws_bytes, f64_main_bytes(m, n, k, s, method))) return rc;
        big = (uint8_t *)dc.ws;
        if (E) CK(cudaEventRecord(E->ev[2], st));
        if (rep) rep->kernel_launches = launches;
        if (int rc = run_main_f64(dev, m, n, k, prec, A, B, C, method, s, bits, st, meta, big, rep, E)) return rc;
        if (rep) {
            rep->slices = s; rep->slice_bits = bits; rep->certified = 1; rep->minT = pb[0]; rep->minT1 = pb[1];
            rep->maxD2 = pb[2]; rep->log2_rho_hat = log2rho;
        }
        if (E) {
            CK(cudaEventSynchronize(E->ev[5]));
            float t[5];
            for (int q = 0; q < 5; q++) CK(cudaEventElapsedTime(&t[q], E->ev[q], E->ev[q + 1]));
            if (rep) { rep->ms_linemax = t[0]; rep->ms_prepass = t[1]; rep->ms_split = t[2]; rep->ms_gemm = t[3]; rep->ms_fold = t[4]; }
        }
        return 0;
    }
    // workspace of row groups of mg rows (the ragged last group may need more slots)
    auto grouped_layout = [&](int64_t mg) {
        const Geometry gg = main_geometry(dev, mg, n, k, s, method, m);
        Layout Lg = layout_for(mg, n, k, s, method, gg.maxkb, prec, beta != 0, gg.g2);
        if (mg < m && m % mg) {
            const int64_t ml = m % mg;
            const int parts = method == 3 ? 3 : 2;
            const Geometry gl = main_geometry(dev, ml, n, k, s, method, m);
            Layout Ll = layout_for(ml, n, k, s, method, gl.maxkb, prec, beta != 0, gl.g2);
            const size_t extra = align_up((size_t)parts * s * mg * Lg.kp, 256) - align_up((size_t)parts * s * ml * Lg.kp, 256);
            Lg.main = std::max(Lg.main, Ll.main + extra);
        }
        return Lg;
    };
    if (group_rows >= m) group_rows = 0;
    // memory bound: when one call's workspace does not fit (the caller's workspace, or free
    // device memory minus 1 GiB, or MPCGEMM_WS_LIMIT bytes), run row groups of 256 * 2^j rows
    size_t budget;
    const size_t want = grouped_layout(group_rows > 0 ? group_rows : m).main;
    if (opts && opts->workspace) budget = opts->workspace_bytes;
    else if (want <= dc.ws_bytes) budget = dc.ws_bytes;          // fits the cached workspace
    else {                                                       // (cudaMemGetInfo costs ~ms)
        size_t fr = 0, tot = 0;
        CK(cudaMemGetInfo(&fr, &tot));
        budget = fr + dc.ws_bytes > ((size_t)1 << 30) ? fr + dc.ws_bytes - ((size_t)1 << 30) : 0;
    }
    if (const char *lim = getenv("MPCGEMM_WS_LIMIT")) if (*lim) budget = std::min(budget, (size_t)strtoull(lim, nullptr, 10));
    if (want > budget) {
        int64_t g = (std::min(group_rows > 0 ? group_rows : m, m) + kSBlk - 1) / kSBlk * kSBlk;
        while (g > kSBlk && grouped_layout(std::min(g, m)).main > budget) g = std::max<int64_t>(kSBlk, g / 2 / kSBlk * kSBlk);
        if (grouped_layout(std::min(g, m)).main > budget) return fail(MPCGEMM_ERR_NOMEM, "workspace for 256-row groups exceeds the budget");
        group_rows = g < m ? g : 0;
    }
    const int64_t mg = group_rows > 0 ? group_rows : m;
    Layout Lm = grouped_layout(mg);
    uint8_t *big;
    if (opts && opts->workspace) {
        if (opts->workspace_bytes < Lm.main) return fail(MPCGEMM_ERR_NOMEM, "caller workspace too small");
        big = (uint8_t *)opts->workspace;
    } else {
        if (int rc = grow(&dc.ws, &dc.ws_bytes, Lm.main)) return rc;
        big = (uint8_t *)dc.ws;
    }
    if (E) CK(cudaEventRecord(E->ev[2], st));
    if (rep) rep->kernel_launches = launches;
    unsigned long long *mma_dev = nullptr;             // device-side MMA count (timed calls)
    if (E && rep) {
        if (!dc.mma_dev) CK(cudaMalloc(&dc.mma_dev, sizeof(unsigned long long)));
        mma_dev = dc.mma_dev;
        CK(cudaMemsetAsync(mma_dev, 0, sizeof(unsigned long long), st));
    }
    if (int rc = run_main(dev, m, n, k, prec, A, B, C, method, s, st, meta, big, Lm, simt, rep, E, beta, alpha_neg,
                          sblk, group_rows, hook, mma_dev))
        return rc;
    if (rep) {
        rep->slices = s; rep->slice_bits = 8; rep->certified = 1; rep->minT = pb[0]; rep->minT1 = pb[1];
        rep->maxD2 = pb[2]; rep->log2_rho_hat = log2rho;
        rep->slices_min = sblk.empty() ? s : *std::min_element(sblk.begin(), sblk.end());
    }
    if (E) {
        CK(cudaEventSynchronize(E->ev[5]));
        float t[5];
        for (int q = 0; q < 5; q++) CK(cudaEventElapsedTime(&t[q], E->ev[q], E->ev[q + 1]));
        if (rep) { rep->ms_linemax = t[0]; rep->ms_prepass = t[1]; rep->ms_split = t[2]; rep->ms_gemm = t[3]; rep->ms_fold = t[4]; }
        if (rep && mma_dev && !simt) {
            unsigned long long h = 0;
            if (int rc = readback(dev, &h, mma_dev, sizeof(h), st)) return rc;
            rep->mma_issued = (int64_t)h;
        }
    }
    return 0;
}

// ---------------------------------------------------------------- NEXT-3: complex LU
mpc_rmat sub_view(const mpc_rmat &M, int64_t r, int64_t c, int L) {
    mpc_rmat v = M;
    const int64_t i = r * M.ld + c;
    v.sign = M.sign + i; v.exp = M.exp + i; v.limbs = M.limbs + i * L;
    return v;
}

// LU factor / solve: one at a time per process (they share the device's LU scratch), and their
// device work ordered after the previous call's like every other call (StreamOrder); g_mu is
// taken only briefly here because the LU's own GEMM updates take it.
std::mutex g_lu_mu;
struct LuOrder {
    int dev; cudaStream_t st;
    LuOrder(int d, cudaStream_t s) : dev(d), st(s) {
        std::lock_guard<std::mutex> lock(g_mu);
        DevCache &dc = g_cache[dev];
        if (dc.done) cudaStreamWaitEvent(st, dc.done, 0);
    }
    ~LuOrder() {
        std::lock_guard<std::mutex> lock(g_mu);
        DevCache &dc = g_cache[dev];
        if (!dc.done) cudaEventCreateWithFlags(&dc.done, cudaEventDisableTiming);
        cudaEventRecord(dc.done, st);
    }
};

int lu_scratch(int dev, int L, LuScratch *s, int32_t **info) {
    std::lock_guard<std::mutex> lock(g_mu);
    DevCache &dc = g_cache[dev];
    if (int rc = grow(&dc.lu, &dc.lu_bytes, 256 + 16 * 2 * (size_t)L + 64)) return rc;
    uint8_t *b = (uint8_t *)dc.lu;
    s->exp = (int64_t *)b; s->limbs = (uint64_t *)(b + 64); s->sign = b + 64 + 16 * 2 * (size_t)L;
    *info = (int32_t *)(b + 64 + 16 * 2 * (size_t)L + 16);
    return 0;
}

struct PhaseTimer {                                     // opts->timing: per-phase CUDA events
    cudaEvent_t a = nullptr, b = nullptr; cudaStream_t st; bool on;
    PhaseTimer(bool on_, cudaStream_t s) : st(s), on(on_) {
        if (on) { cudaEventCreate(&a); cudaEventCreate(&b); cudaEventRecord(a, st); }
    }
    ~PhaseTimer() { if (a) cudaEventDestroy(a); if (b) cudaEventDestroy(b); }
    void lap(float *acc) {
        if (!on) return;
        float ms = 0.f;
        cudaEventRecord(b, st); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        *acc += ms; std::swap(a, b);
    }
};

int lu_impl(int64_t n, int32_t prec, mpc_cmat *A, int64_t *ipiv, int32_t K, int method, const mpcgemm_opts *opts,
            mpclu_report *rep) {
    if (rep) memset(rep, 0, sizeof(*rep));
    if (!A || !ipiv || n < 0 || K < 1) return fail(MPCGEMM_ERR_ARG, "mpclu_factor: bad argument");
    if (method != MPCGEMM_3M && method != MPCGEMM_4M) return fail(MPCGEMM_ERR_ARG, "method must be 3 or 4");
    if (prec < 2 || prec > 1024) return fail(MPCGEMM_ERR_PREC, "mpclu_factor: prec outside [2, 1024]");
    if (n == 0) return 0;
    if (A->re.ld < n || A->im.ld < n || !A->re.sign || !A->im.sign) return fail(MPCGEMM_ERR_ARG, "mpclu_factor: bad matrix");
    const int L = (prec + 63) / 64;
    cudaStream_t st = opts ? (cudaStream_t)opts->stream : nullptr;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lulock(g_lu_mu);
    LuOrder order(dev, st);
    LuScratch sc; int32_t *info;
    if (int rc = lu_scratch(dev, L, &sc, &info)) return rc;
    CK(cudaMemsetAsync(info, 0, 4, st));
    const DMatOut re = dmo(A->re), im = dmo(A->im);
    PhaseTimer T(opts && opts->timing, st);
    float tp = 0.f, tt = 0.f, tg = 0.f;
    int launches = 0, calls = 0, smax = 0;
    for (int64_t j0 = 0; j0 < n; j0 += K) {
        const int64_t w = std::min<int64_t>(K, n - j0);
        for (int64_t c = j0; c < j0 + w; c++) {               // (a) panel, xGETF2
            CK(lu_pivot_launch(L, re, im, n, c, ipiv, st));
            CK(lu_swap_launch(L, re, im, n, c, ipiv, st));
            int nrs = 0;
            CK(lu_recip_scale_launch(L, re, im, c + 1, n, c, prec, sc, info, &nrs, st));
            CK(lu_update_launch(L, re, im, c + 1, n, c + 1, j0 + w, c, prec, st));
            launches += 3 + nrs;
        }
        T.lap(&tp);
        if (j0 + w >= n) break;
        for (int64_t c = j0; c < j0 + w - 1; c++) {           // (b) U12 := L11^-1 A12
            CK(lu_update_launch(L, re, im, c + 1, j0 + w, j0 + w, n, c, prec, st));
            launches++;
        }
        T.lap(&tt);
        const int64_t m2 = n - j0 - w;                        // (c) A22 -= L21 U12 (Ozaki)
        mpc_cmat L21{sub_view(A->re, j0 + w, j0, L), sub_view(A->im, j0 + w, j0, L)};
        mpc_cmat U12{sub_view(A->re, j0, j0 + w, L), sub_view(A->im, j0, j0 + w, L)};
        mpc_cmat A22{sub_view(A->re, j0 + w, j0 + w, L), sub_view(A->im, j0 + w, j0 + w, L)};
        mpcgemm_opts o;
        memset(&o, 0, sizeof(o));
        o.stream = (void *)st; o.beta = 1; o.alpha_neg = 1; o.adaptive = opts ? opts->adaptive : 0;
        mpcgemm_report gr;
        if (int rc = gemm_impl(m2, m2, w, prec, &L21, &U12, &A22, method, &o, &gr, false)) { if (rc < 0) return rc; }
        smax = std::max(smax, gr.slices);
        launches += gr.kernel_launches;
        calls++;
        T.lap(&tg);
    }
    int32_t h = 0;
    CK(cudaMemcpyAsync(&h, info, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (rep) {
        rep->info = h; rep->gemm_calls = calls; rep->slices_max = smax; rep->kernel_launches = launches;
        rep->ms_panel = tp; rep->ms_trsm = tt; rep->ms_gemm = tg;
    }
    return 0;
}

}  // namespace

// ================================================================== C ABI
extern "C" {

int mpcgemm(int64_t m, int64_t n, int64_t k, int32_t prec, const mpc_cmat *A, const mpc_cmat *B, mpc_cmat *C,
            mpcgemm_method method) {
    return gemm_impl(m, n, k, prec, A, B, C, (int)method, nullptr, nullptr);
}

int mpcgemm_ex(int64_t m, int64_t n, int64_t k, int32_t prec, const mpc_cmat *A, const mpc_cmat *B, mpc_cmat *C,
               mpcgemm_method method, const mpcgemm_opts *opts, mpcgemm_report *rep) {
    return gemm_impl(m, n, k, prec, A, B, C, (int)method, opts, rep);
}

int mpcgemm_rho_bounds(int64_t m, int64_t n, int64_t k, int32_t prec, const mpc_cmat *A, const mpc_cmat *B,
                       int32_t full, const mpcgemm_opts *opts, int64_t out[3]) {
    if (!out) return fail(MPCGEMM_ERR_ARG, "null out");
    if (!A || !B) return fail(MPCGEMM_ERR_ARG, "null matrix descriptor");
    if (m < 0 || n < 0 || k < 0) return fail(MPCGEMM_ERR_ARG, "negative dimension");
    if (prec < 2 || prec > 4096) return fail(MPCGEMM_ERR_PREC, "prec outside [2, 4096]");
    out[0] = out[1] = out[2] = -1;
    if (m == 0 || n == 0 || k == 0) return 0;
    cudaStream_t st = opts ? (cudaStream_t)opts->stream : nullptr;
    const int L = (prec + 63) / 64;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(g_mu);
    DevCache &dc = g_cache[dev];
    StreamOrder order(dc, st);
    Layout Lo = layout_for(m, n, k, 0, MPCGEMM_3M, kMaxKBlocksPerChunk);
    if (int rc = grow(&dc.meta, &dc.meta_bytes, Lo.meta)) return rc;
    if (int rc = grow(&dc.ws, &dc.ws_bytes, Lo.pre)) return rc;
    uint8_t *meta = (uint8_t *)dc.meta;
    const MetaView mv = meta_view(meta, m, n);
    CK(linemax2_launch(dm(A->re), dm(A->im), dm(B->re), dm(B->im), m, n, k, L, prec, mv.eA, mv.nzA, nullptr, 0, st));
    Bounds bd;
    if (int rc = run_prepass(dev, m, n, k, prec, A, B, full, st, meta, (uint8_t *)dc.ws, Lo,
                             env_int("MPCGEMM_SLICEGEMM_SIMT", 0), &bd))
        return rc;
    for (int q = 0; q < 3; q++) out[q] = bd.g[q];
    return 0;
}

int mpcgemm_slices_for(int32_t prec, mpcgemm_method method, int64_t k, int64_t minT, int64_t minT1, int64_t maxD2) {
    return rule_slices(prec, (int)method, rule_log2rho(k, minT, minT1, maxD2));
}

size_t mpcgemm_workspace_size(int64_t m, int64_t n, int64_t k, int32_t prec, mpcgemm_method method, int32_t slices) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (slices <= 0) {                                 // auto: the s of the rule at minT = 1, the
        slices = rule_slices(prec, (int)method, rule_log2rho(std::max<int64_t>(k, 1), 1, 1, -1));   // largest
        if (slices < 0) slices = kMaxSlices;           // first-stage s (max-plus inputs may need more)
    }
    const Geometry gw = main_geometry(dev, m, n, k, slices, (int)method);
    Layout Lo = layout_for(m, n, k, slices, (int)method, gw.maxkb, prec, true, gw.g2);
    return std::max(Lo.main, Lo.pre);
}

// e2e entry: H2D of A, B (and C0), the hot path in row groups, and the D2H of each finished
// group of C on a second stream while the next group computes (MPCGEMM_HOST_GROUP rows per
// group, a multiple of 256; default 512 when m >= 1024; 0 = one group)
std::mutex g_host_mu;                                  // one host-buffer call at a time (staging)

// e2e entry (sync: returns with C on the host; async: returns once the call's device work is
// queued -- H2D on the h2d stream into staging set j, compute on st, D2H of finished row groups
// on the copy stream -- and set j is released by an event when its D2H is done)
int host_impl(int64_t m, int64_t n, int64_t k, int32_t prec, const mpc_cmat *A, const mpc_cmat *B, mpc_cmat *C,
              mpcgemm_method method, const mpcgemm_opts *opts, mpcgemm_report *rep, bool async) {
    if (int rc = check_args(m, n, k, prec, A, B, C, (int)method)) return rc;
    std::lock_guard<std::mutex> hostlock(g_host_mu);
    const int L = (prec + 63) / 64;
    cudaStream_t st = opts ? (cudaStream_t)opts->stream : nullptr;
    const mpc_rmat *in[4] = {&A->re, &A->im, &B->re, &B->im};
    const int64_t rows[6] = {m, m, k, k, m, m}, cols[6] = {k, k, n, n, n, n};
    size_t off[6][3], total = 0;
    for (int q = 0; q < 6; q++) {
        const size_t ents = (size_t)rows[q] * cols[q];
        off[q][0] = total; total = align_up(total + ents, 256);
        off[q][1] = total; total = align_up(total + ents * 8, 256);
        off[q][2] = total; total = align_up(total + ents * 8 * L, 256);
    }
    int dev = 0;
    CK(cudaGetDevice(&dev));
    uint8_t *base;
    cudaStream_t cs, hs;                               // D2H copy stream, H2D stream
    cudaEvent_t ev, ev_in, ev_free;
    {
        std::lock_guard<std::mutex> lock(g_mu);
        DevCache &dc = g_cache[dev];
        if (!dc.copy_stream) {
            CK(cudaStreamCreateWithFlags(&dc.copy_stream, cudaStreamNonBlocking));
            CK(cudaStreamCreateWithFlags(&dc.h2d_stream, cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&dc.group_event, cudaEventDisableTiming));
            for (int j = 0; j < 2; j++) {
                CK(cudaEventCreateWithFlags(&dc.stage_in[j], cudaEventDisableTiming));
                CK(cudaEventCreateWithFlags(&dc.stage_free[j], cudaEventDisableTiming));
            }
        }
        const int j = async ? dc.stage_next : 0;       // sync calls keep to set 0 (one set of memory)
        if (async) dc.stage_next ^= 1;
        if (int rc = grow(&dc.stage[j], &dc.stage_bytes[j], total)) return rc;   // grow syncs before a free
        base = (uint8_t *)dc.stage[j];
        cs = dc.copy_stream; hs = dc.h2d_stream; ev = dc.group_event;
        ev_in = dc.stage_in[j]; ev_free = dc.stage_free[j];
    }
    mpc_rmat dmats[6];
    for (int q = 0; q < 6; q++) {
        dmats[q].sign = base + off[q][0];
        dmats[q].exp = (int64_t *)(base + off[q][1]);
        dmats[q].limbs = (uint64_t *)(base + off[q][2]);
        dmats[q].ld = cols[q];
    }
    // the H2D waits until the set's previous call has finished with it (its D2H included)
    CK(cudaStreamWaitEvent(hs, ev_free, 0));
    for (int q = 0; q < 4; q++) {
        const mpc_rmat &H = *in[q];
        if (rows[q] == 0 || cols[q] == 0) continue;
        CK(cudaMemcpy2DAsync(dmats[q].sign, cols[q], H.sign, H.ld, cols[q], rows[q], cudaMemcpyHostToDevice, hs));
        CK(cudaMemcpy2DAsync(dmats[q].exp, cols[q] * 8, H.exp, H.ld * 8, cols[q] * 8, rows[q], cudaMemcpyHostToDevice, hs));
        CK(cudaMemcpy2DAsync(dmats[q].limbs, cols[q] * 8 * L, H.limbs, H.ld * 8 * L, cols[q] * 8 * L, rows[q],
                             cudaMemcpyHostToDevice, hs));
    }
    if (opts && opts->beta) {                          // C is an input too
        const mpc_rmat *cin[2] = {&C->re, &C->im};
        for (int q = 0; q < 2; q++) {
            if (m == 0 || n == 0) continue;
            const mpc_rmat &H = *cin[q];
            CK(cudaMemcpy2DAsync(dmats[4 + q].sign, n, H.sign, H.ld, n, m, cudaMemcpyHostToDevice, hs));
            CK(cudaMemcpy2DAsync(dmats[4 + q].exp, n * 8, H.exp, H.ld * 8, n * 8, m, cudaMemcpyHostToDevice, hs));
            CK(cudaMemcpy2DAsync(dmats[4 + q].limbs, n * 8 * L, H.limbs, H.ld * 8 * L, n * 8 * L, m,
                                 cudaMemcpyHostToDevice, hs));
        }
    }
    CK(cudaEventRecord(ev_in, hs));
    CK(cudaStreamWaitEvent(st, ev_in, 0));
    mpc_cmat dA{dmats[0], dmats[1]}, dB{dmats[2], dmats[3]}, dC{dmats[4], dmats[5]};
    mpc_rmat *outs[2] = {&C->re, &C->im};
    // D2H of C rows [r0, r1) on the copy stream once the compute stream has finished them
    GroupHook d2h = [&](int64_t r0, int64_t r1) -> int {
        if (n == 0 || r1 <= r0) return 0;
        CK(cudaEventRecord(ev, st));
        CK(cudaStreamWaitEvent(cs, ev, 0));
        for (int q = 0; q < 2; q++) {
            const mpc_rmat &D = dmats[4 + q];
            mpc_rmat &H = *outs[q];
            const int64_t nr = r1 - r0;
            CK(cudaMemcpy2DAsync(H.sign + r0 * H.ld, H.ld, D.sign + r0 * n, n, n, nr, cudaMemcpyDeviceToHost, cs));
            CK(cudaMemcpy2DAsync(H.exp + r0 * H.ld, H.ld * 8, D.exp + r0 * n, n * 8, n * 8, nr, cudaMemcpyDeviceToHost, cs));
            CK(cudaMemcpy2DAsync(H.limbs + r0 * H.ld * L, H.ld * 8 * L, D.limbs + r0 * n * L, n * 8 * L, n * 8 * L, nr,
                                 cudaMemcpyDeviceToHost, cs));
        }
        return 0;
    };
    // row groups let a blocking call's D2H overlap its own later groups (~7 ms of extra GEMM
    // tails and B re-reads at config 4); a queued call's D2H overlaps the next call instead
    int64_t group = env_int("MPCGEMM_HOST_GROUP", (!async && m >= 1024) ? 512 : 0);
    if (group > 0) group = std::max<int64_t>(kSBlk, group / kSBlk * kSBlk);
    const bool grouped = group > 0 && group < m && !(opts && opts->carrier == 1);
    int rc = gemm_impl(m, n, k, prec, &dA, &dB, &dC, (int)method, opts, rep, true, grouped ? group : 0,
                       grouped ? &d2h : nullptr);
    if (rc >= 0 && !grouped) {
        if (int r2 = d2h(0, m)) rc = r2;
    }
    // the set is free once everything queued for this call has run (compute and D2H)
    CK(cudaEventRecord(ev, st));
    CK(cudaStreamWaitEvent(cs, ev, 0));
    CK(cudaEventRecord(ev_free, cs));
    if (rc < 0 || !async) {
        CK(cudaStreamSynchronize(st));
        CK(cudaStreamSynchronize(cs));
    }
    return rc;
}

int mpcgemm_host(int64_t m, int64_t n, int64_t k, int32_t prec, const mpc_cmat *A, const mpc_cmat *B, mpc_cmat *C,
                 mpcgemm_method method, const mpcgemm_opts *opts, mpcgemm_report *rep) {
    return host_impl(m, n, k, prec, A, B, C, method, opts, rep, false);
}

int mpcgemm_host_async(int64_t m, int64_t n, int64_t k, int32_t prec, const mpc_cmat *A, const mpc_cmat *B,
                       mpc_cmat *C, mpcgemm_method method, const mpcgemm_opts *opts, mpcgemm_report *rep) {
    return host_impl(m, n, k, prec, A, B, C, method, opts, rep, true);
}

int mpcgemm_host_wait(void) {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    cudaEvent_t fr[2] = {};
    {
        std::lock_guard<std::mutex> lock(g_mu);
        auto it = g_cache.find(dev);
        if (it == g_cache.end() || !it->second.copy_stream) return 0;
        fr[0] = it->second.stage_free[0]; fr[1] = it->second.stage_free[1];
    }
    for (int j = 0; j < 2; j++) CK(cudaEventSynchronize(fr[j]));
    CK(cudaGetLastError());
    return 0;
}

int mpcgemm_device_rule_result(int64_t m, int64_t n, void *stream, int64_t out[4]) {
    if (!out) return fail(MPCGEMM_ERR_ARG, "null out");
    int dev = 0;
    CK(cudaGetDevice(&dev));
    cudaStream_t st = (cudaStream_t)stream;
    std::lock_guard<std::mutex> lock(g_mu);
    DevCache &dc = g_cache[dev];
    if (!dc.meta || dc.meta_bytes < meta_bytes(m, n)) return fail(MPCGEMM_ERR_ARG, "no device-rule call of this shape");
    const MetaView mv = meta_view((uint8_t *)dc.meta, m, n);
    DevRuleState h;
    if (int rc = readback(dev, &h, mv.drs, sizeof(h), st)) return rc;
    out[0] = h.s_needed; out[1] = h.minT; out[2] = h.minT1; out[3] = h.maxD2;
    return h.status;
}

const char *mpcgemm_strerror(int code) {
    switch (code) {
        case MPCGEMM_OK: return "ok";
        case MPCGEMM_ERR_ARG: return "invalid argument";
        case MPCGEMM_ERR_PREC: return "precision outside [2, 4096]";
        case MPCGEMM_ERR_EXP_RANGE: return "exponent outside [-2^61, 2^61]";
        case MPCGEMM_ERR_NOT_NORMALIZED: return "mantissa not normalized";
        case MPCGEMM_ERR_ALIAS: return "C overlaps A or B";
        case MPCGEMM_ERR_NOMEM: return "workspace allocation failed";
        case MPCGEMM_ERR_CUDA: return "CUDA error";
        case MPCGEMM_ERR_SLICES: return "slice count outside [1, 1024]";
        default: return "unknown status";
    }
}

const char *mpcgemm_last_error(void) { return g_last_error.c_str(); }

void mpcgemm_release(void) {
    std::lock_guard<std::mutex> lock(g_mu);
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return;
    cudaDeviceSynchronize();
    auto it = g_cache.find(dev);
    if (it != g_cache.end()) {
        if (it->second.done) cudaEventDestroy(it->second.done);
        cudaFree(it->second.ws); cudaFree(it->second.meta); cudaFree(it->second.stage[0]); cudaFree(it->second.stage[1]);
        cudaFree(it->second.lu); cudaFree(it->second.lm); cudaFree(it->second.tb);
        cudaFree(it->second.solve);
        cudaFree(it->second.mma_dev);
        if (it->second.rb) cudaFreeHost(it->second.rb);
        g_cache.erase(it);
    }
    for (auto p = g_devplans.begin(); p != g_devplans.end();) {
        if (std::get<0>(p->first) == dev) { cudaFree(p->second.d_plans); cudaFree(p->second.d_counter); p = g_devplans.erase(p); }
        else ++p;
    }
    for (auto p = g_plans.begin(); p != g_plans.end();) {
        if (p->first.first == dev) {
            cudaFree(p->second.d_units); cudaFree(p->second.d_counter); cudaFree(p->second.d_slotinfo);
            p = g_plans.erase(p);
        } else ++p;
    }
}

int mpclu_factor(int64_t n, int32_t prec, mpc_cmat *A, int64_t *ipiv, int32_t K, mpcgemm_method method,
                 const mpcgemm_opts *opts, mpclu_report *rep) {
    return lu_impl(n, prec, A, ipiv, K, (int)method, opts, rep);
}

int mpclu_solve(int64_t n, int64_t nrhs, int32_t prec, const mpc_cmat *LU, const int64_t *ipiv, mpc_cmat *B,
                const mpcgemm_opts *opts) {
    if (!LU || !ipiv || !B || n < 0 || nrhs < 0) return fail(MPCGEMM_ERR_ARG, "mpclu_solve: bad argument");
    if (prec < 2 || prec > 1024) return fail(MPCGEMM_ERR_PREC, "mpclu_solve: prec outside [2, 1024]");
    if (n == 0 || nrhs == 0) return 0;
    if (LU->re.ld < n || LU->im.ld < n || B->re.ld < nrhs || B->im.ld < nrhs) return fail(MPCGEMM_ERR_ARG, "mpclu_solve: ld");
    const int L = (prec + 63) / 64;
    cudaStream_t st = opts ? (cudaStream_t)opts->stream : nullptr;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lulock(g_lu_mu);
    LuOrder order(dev, st);
    // scratch: 1 x n reciprocals and the n x nrhs solution, both parts (ABI element format)
    const size_t ents = (size_t)n + (size_t)n * nrhs;
    uint8_t *base;
    {
        std::lock_guard<std::mutex> lock(g_mu);
        DevCache &dc = g_cache[dev];
        if (int rc = grow(&dc.solve, &dc.solve_bytes, 2 * ents * (9 + 8 * (size_t)L) + 8 * (size_t)n + 8192)) return rc;
        base = (uint8_t *)dc.solve;
    }
    auto carve = [&](size_t cnt, int64_t ldm) {
        DMatOut M;
        M.limbs = (uint64_t *)base; base += align_up(cnt * 8 * L, 256);
        M.exp = (int64_t *)base; base += align_up(cnt * 8, 256);
        M.sign = base; base += align_up(cnt, 256);
        M.ld = ldm;
        return M;
    };
    SolveScratch sc;
    sc.rre = carve(n, n); sc.rim = carve(n, n);
    sc.xre = carve((size_t)n * nrhs, nrhs); sc.xim = carve((size_t)n * nrhs, nrhs);
    sc.perm = (int64_t *)base;
    CK(lu_solve_launch(L, dmo(LU->re), dmo(LU->im), n, ipiv, dmo(B->re), dmo(B->im), nrhs, prec, sc, st));
    return 0;
}

int mpc_scalar(int32_t op, int64_t cnt, int32_t prec, const mpc_cmat *A, const mpc_cmat *X, const mpc_cmat *Y,
               mpc_cmat *O, int64_t *kv, void *stream) {
    if (op < 0 || op > 3 || cnt < 0 || !X) return fail(MPCGEMM_ERR_ARG, "mpc_scalar: bad argument");
    if (prec < 2 || prec > 1024) return fail(MPCGEMM_ERR_PREC, "mpc_scalar: prec outside [2, 1024]");
    if ((op == 3 && !kv) || (op != 3 && !O) || ((op == 0 || op == 1) && !Y) || (op == 1 && !A))
        return fail(MPCGEMM_ERR_ARG, "mpc_scalar: missing operand");
    const int L = (prec + 63) / 64;
    const mpc_cmat *a = A ? A : X, *y = Y ? Y : X;
    const mpc_cmat *o = O ? O : X;
    CK(mp_scalar_launch(L, op, cnt, prec, dmo(a->re), dmo(a->im), dmo(X->re), dmo(X->im), dmo(y->re), dmo(y->im),
                        dmo(o->re), dmo(o->im), kv, (cudaStream_t)stream));
    return 0;
}

int mpcgemm_version(void) { return 100; }

}  // extern "C"
