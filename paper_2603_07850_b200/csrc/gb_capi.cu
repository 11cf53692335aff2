// gb_capi.cu -- implementation of the C-ABI boundary (include/goldbach_b200.h).
//
// One gb_dev per GPU.  Segments submitted by the host worker are cut into
// device pieces (<= 2^31 evens), packed S per batch, and each batch runs
// as one stream of kernels:
//   H2D jobs -> [large-prime strike] -> segment offsets -> fused sieve+check
//   -> stragglers/Phase 2 -> finalize -> D2H records
// Up to NBATCH batches are in flight on separate streams so the tail of one
// fused launch overlaps the head of the next.  Nothing here computes on the
// CPU: host code only schedules, copies records and merges them
// (MinPrimeMax / sums / counterexample lists, pool.cpp:159-174 semantics).
#include <algorithm>
#include <dlfcn.h>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <mutex>
#include <string>
#include <vector>

#include "gb_arena.h"
#include "gb_kernels.h"

using namespace gbk;

namespace {

constexpr int NBATCH = 3;                 // batches in flight per device
constexpr uint32_t SLOTS = MAX_SLOTS;     // pieces per batch
constexpr uint32_t LIST_CAP = 1u << 20;   // straggler entries per batch
constexpr uint64_t MAX_PIECE = MAX_SEG_EVENS; // cells of a piece stay < 2^31 - 1 (block_off)

thread_local std::string t_err;

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

uint64_t sqrt_bound_of(uint64_t cover) {
    // build_base_primes' s (sieve.cpp:48-52): minimal s with s >= cover / s
    uint64_t s = (uint64_t)std::sqrt((long double)cover);
    if (s == 0) s = 1;
    while (s > 1 && (s - 1) >= cover / (s - 1)) --s;
    while (s < cover / s) ++s;
    return s;
}

uint64_t isqrt_floor(uint64_t x) {
    uint64_t r = (uint64_t)std::sqrt((long double)x);
    while (r > 0 && r > x / r) --r;
    while ((r + 1) <= x / (r + 1)) ++r;
    return r;
}

struct Piece {
    uint64_t seq; // user segment sequence number
    uint64_t a, b;
};

struct Batch {
    cudaStream_t st = nullptr;
    SegJob* d_jobs = nullptr;
    uint4* d_pmc = nullptr;           // per slot {p, magic, c0} of the tile primes
    uint32_t* d_qg = nullptr;
    uint32_t* d_k00 = nullptr;          // per-batch first indices of the primes > P_TILE_MAX (k_large_first)
    SlotAcc* d_acc = nullptr;
    StragEntry* d_list = nullptr;
    unsigned int* d_counters = nullptr; // [0] block counter, [1] list count
    StragResult* d_res = nullptr;
    DevRecord* d_rec = nullptr;
    SegJob* h_jobs = nullptr;
    DevRecord* h_rec = nullptr;
    cudaEvent_t ev_done = nullptr, ev_k0 = nullptr, ev_k1 = nullptr, ev_l0 = nullptr, ev_s1 = nullptr;
    cudaEvent_t ev_first = nullptr;     // after the large-prime launches (k00 written; gb_dev::chain_b)
    std::vector<Piece> pieces;
    bool launched = false;
    bool timed = false;
    bool pre = false;                   // pre-kernels timed (mask fill / large strike)
};

struct UserSeg {
    uint64_t seq, a, b, tag;
    uint32_t pieces_total = 0, pieces_done = 0;
    gb_seg_record rec{};
    double t0 = 0;
};

} // namespace

struct gb_dev {
    int device = 0;
    gb_params prm{};
    std::string err;
    int sms = 148, occ = 2;
    uint64_t sqrt_bound = 0, n_primes = 0;
    uint32_t* d_primes = nullptr;
    uint32_t iA0 = 0, iA1 = 0, iB1 = 0; // tile prime index ranges
    uint32_t iQ1 = 0, iH1 = 0;          // first tile primes >= M6/4, >= M6/2
    uint32_t iW1 = 0;                   // first tile prime >= W
    uint16_t* d_wsplit = nullptr;       // [SPLIT_WARPS][32] balanced warp-cooperative primes (light split)
    uint16_t* d_wsplit_heavy = nullptr; // the same for the heavy split
    uint16_t* d_wsplit_mask = nullptr;  // and for the mask split
    uint64_t* d_m64 = nullptr;          // floor(2^64 / p) per base prime
    uint32_t* d_m32 = nullptr;          // floor(2^32 / p) per prime > P_TILE_MAX (GB_LS_PRE=0: none)
    uint64_t iL0 = 0, iL1 = 0;          // large primes
    uint64_t iLB = 0;                   // first large prime of the batch walk (k_large_batch); iL1 = none
    uint32_t ls_cop = 0;                // k_large_rows skips multiples of 5..13 (1) and 17..23 (2) (GB_LS_COP; default 0: measured slower)
    Batch* chain_b = nullptr;           // batch whose k00 buffer holds the last row walk's first indices
    Batch* last_large = nullptr;        // batch of the last large-prime launches (ev_first orders the next)
    uint64_t chain_q0 = 0;              // ... and its slot-0 origin (|Q|, positive)
    bool ls_chain = false;              // derive k00 from chain_b's (GB_LS_CHAIN=1; off: measured neutral, C5 0.142 s on against 0.140-0.141 s off)
    bool ls_rows = true;                // row walk (k_large_rows) for batches on one axis (GB_LS_ROWS=0: per slot)
    // mask fill (k_mask_fill): tile primes [iK0, iB1) struck per 3-block
    // range into the large-prime bitmask instead of visited by every block
    bool mk_on = false;                 // plan built
    bool mk_off_now = false;            // rows only (gb_set_bucket(dev, 0))
    uint32_t iK0 = 0;
    uint32_t mk_p0 = 0;                 // smallest mask prime
    uint32_t force_sw = 0;              // GB_SW: force a compiled split (tuning)
    bool pair = false;                  // GB_PAIR=1: k_verify_pair (2-CTA clusters share the single-strike rows)
    uint32_t* d_pat = nullptr;
    uint32_t* d_pat6 = nullptr;         // wheel-6 presieve patterns
    uint64_t* d_masks6 = nullptr;       // wheel-6 deep-window masks
    uint64_t max_piece = 0;
    uint64_t qg_stride = 0; // words per slot
    Batch batches[NBATCH];
    int fill = -1;                 // batch being filled
    std::deque<int> inflight;      // launched batches, oldest first
    std::deque<UserSeg> segs;      // submitted user segments, FIFO
    uint64_t next_seq = 0;
    uint64_t launches = 0;
    bool timing = false;
    bool serial = false;           // timing mode 2: every batch on one stream
    uint64_t h2d_bytes = 0, d2h_bytes = 0;
    void* flush_buf = nullptr;
    double kms[4] = {0, 0, 0, 0};
    uint64_t kl[4] = {0, 0, 0, 0};
    Batch sync;                    // private batch for the synchronous helpers
    cudaEvent_t tm0 = nullptr, tm1 = nullptr; // gb_device_timer
    cudaEvent_t t_ref = nullptr;   // timing origin (gb_set_timing)
    double last_k1 = 0;            // end of the last fused launch, ms after t_ref
};

#define GB_FAIL(dev, code, msg)                      \
    do {                                             \
        set_err(dev, msg);                           \
        return code;                                 \
    } while (0)

#define CU(dev, expr)                                                                      \
    do {                                                                                   \
        cudaError_t _e = (expr);                                                           \
        if (_e != cudaSuccess) {                                                           \
            set_err(dev, std::string(#expr) + ": " + cudaGetErrorString(_e));              \
            return GB_ERR_CUDA;                                                            \
        }                                                                                  \
    } while (0)

static void set_err(gb_dev* d, const std::string& m) {
    if (d) d->err = m;
    t_err = m;
}

// --------------------------------------------------------------- batches
static int batch_alloc(gb_dev* d, Batch& b, bool with_qg) {
    if (!b.st) CU(d, cudaStreamCreateWithFlags(&b.st, cudaStreamNonBlocking));
    uint32_t np = d->iB1 - d->iA0;
    CU(d, dmalloc(d->device, &b.d_jobs, SLOTS * sizeof(SegJob)));
    CU(d, dmalloc(d->device, &b.d_pmc, (size_t)SLOTS * std::max<uint32_t>(np, 1) * sizeof(uint4)));
    if (with_qg && (d->iL1 > d->iL0 || d->mk_on))
        CU(d, dmalloc(d->device, &b.d_qg, (size_t)SLOTS * d->qg_stride * 4));
    if (with_qg && d->d_m32) CU(d, dmalloc(d->device, &b.d_k00, (size_t)(d->iL1 - d->iL0) * 4));
    CU(d, dmalloc(d->device, &b.d_acc, SLOTS * sizeof(SlotAcc)));
    CU(d, dmalloc(d->device, &b.d_list, (size_t)LIST_CAP * sizeof(StragEntry)));
    CU(d, dmalloc(d->device, &b.d_counters, 4 * sizeof(unsigned int)));
    CU(d, dmalloc(d->device, &b.d_res, (size_t)LIST_CAP * sizeof(StragResult)));
    CU(d, dmalloc(d->device, &b.d_rec, SLOTS * sizeof(DevRecord)));
    CU(d, hmalloc(&b.h_jobs, SLOTS * sizeof(SegJob)));
    CU(d, hmalloc(&b.h_rec, SLOTS * sizeof(DevRecord)));
    CU(d, cudaEventCreateWithFlags(&b.ev_done, cudaEventDisableTiming));
    CU(d, cudaEventCreate(&b.ev_k0));
    CU(d, cudaEventCreate(&b.ev_k1));
    CU(d, cudaEventCreate(&b.ev_l0));
    CU(d, cudaEventCreate(&b.ev_s1));
    CU(d, cudaEventCreateWithFlags(&b.ev_first, cudaEventDisableTiming));
    return GB_OK;
}

static void batch_free(gb_dev* d, Batch& b) {
    dfree(d->device, b.d_jobs);
    dfree(d->device, b.d_pmc);
    dfree(d->device, b.d_qg);
    dfree(d->device, b.d_k00);
    dfree(d->device, b.d_acc);
    dfree(d->device, b.d_list);
    dfree(d->device, b.d_counters);
    dfree(d->device, b.d_res);
    dfree(d->device, b.d_rec);
    hfree(b.h_jobs);
    hfree(b.h_rec);
    if (b.ev_done) cudaEventDestroy(b.ev_done);
    if (b.ev_k0) cudaEventDestroy(b.ev_k0);
    if (b.ev_k1) cudaEventDestroy(b.ev_k1);
    if (b.ev_l0) cudaEventDestroy(b.ev_l0);
    if (b.ev_s1) cudaEventDestroy(b.ev_s1);
    if (b.ev_first) cudaEventDestroy(b.ev_first);
    if (b.st) cudaStreamDestroy(b.st);
    b = Batch{};
}

// Fill the job descriptor of one piece: wheel-6 blocks of E6 evens whose
// windows start at Q_b = Q + 6 K6 b, Q = the largest q = 1 (mod 6) with
// q <= a - PH6 (negative near the start of the number line).
static void make_job(gb_dev* d, const Piece& pc, SegJob& j, uint32_t prefix, bool use_qg) {
    j.a = pc.a;
    j.b = pc.b;
    j.evens = (uint32_t)(((pc.b - pc.a) >> 1) + 1);
    j.nblocks = (j.evens + E6 - 1) / E6;
    j.block_prefix = prefix;
    if (pc.a >= PH6 + 1) {
        const uint64_t x = pc.a - PH6; // >= 1
        const uint64_t q = x - ((x - 1) % 6);
        j.qneg = 0;
        j.qbase = q;
        j.delta = (uint32_t)(pc.a - q);
        for (int g = 0; g < 4; ++g) j.qmod[g] = (uint32_t)(q % pg6_p(g));
    } else {
        const int64_t x = (int64_t)pc.a - (int64_t)PH6; // <= 0
        const int64_t q = x - (((x - 1) % 6) + 6) % 6;
        j.qneg = 1;
        j.qbase = (uint64_t)(-q);
        j.delta = (uint32_t)((int64_t)pc.a - q);
        for (int g = 0; g < 4; ++g) {
            const int64_t P = pg6_p(g);
            j.qmod[g] = (uint32_t)(((q % P) + P) % P);
        }
    }
    j.qg_words = use_qg ? (uint32_t)(((uint64_t)j.nblocks * K6 + (M6 - K6) + 31) / 32) : 0;
}

// Slot table of k_large_batch: every slot on slot 0's wheel axis (origin
// Q_0, q = Q_0 + 6k), ascending, the span below 2^32 cells, and each window
// overlapping at most its neighbours' (the halo), so that a cell lies in the
// last slot starting at or below it or in the one before.
static bool large_batch_tab(const SegJob* J, uint32_t n, LargeBatchTab& T) {
    if (n == 0 || n > MAX_SLOTS) return false;
    for (uint32_t s = 0; s < MAX_SLOTS; ++s) T.d[s] = ~0u;
    uint64_t span = 0;
    for (uint32_t s = 0; s < n; ++s) {
        if (J[s].qneg || J[s].qbase < J[0].qbase) return false;
        const uint64_t dd = (J[s].qbase - J[0].qbase) / 6;
        const uint64_t end = dd + (uint64_t)J[s].qg_words * 32;
        if (end >= (1ull << 32) - 1) return false;
        if (s > 0 && dd < T.d[s - 1]) return false;
        if (s > 1 && dd < (uint64_t)T.d[s - 2] + (uint64_t)J[s - 2].qg_words * 32) return false;
        T.d[s] = (uint32_t)dd;
        T.qw[s] = J[s].qg_words;
        T.qm[s][0] = (uint32_t)(J[s].qbase % 5005);
        T.qm[s][1] = (uint32_t)((J[s].qbase % 5005 + 4) % 5005);
        T.qm2[s][0] = (uint32_t)(J[s].qbase % 7429);
        T.qm2[s][1] = (uint32_t)((J[s].qbase % 7429 + 4) % 7429);
        span = std::max(span, end);
    }
    // k_large_rows forms 6 o + (origin mod 7429) for o below a row's span
    for (uint32_t s = 0; s < n; s += 2) {
        const uint64_t e0 = (uint64_t)J[s].qg_words * 32;
        const uint64_t e1 = s + 1 < n ? (uint64_t)(T.d[s + 1] - T.d[s]) + (uint64_t)J[s + 1].qg_words * 32 : 0;
        if (6 * std::max(e0, e1) + 7429 >= (1ull << 32)) return false;
    }
    T.n = n;
    T.span = (uint32_t)span;
    return true;
}

static int batch_launch(gb_dev* d, Batch& b, uint64_t* pmin_out, uint32_t* tile_out = nullptr,
                        uint32_t tile_fb = 0) {
    const uint32_t n = (uint32_t)b.pieces.size();
    const bool large = d->iL1 > d->iL0;          // primes > P_TILE_MAX: k_large_strike
    const bool mask = d->mk_on && !d->mk_off_now; // tile primes >= iK0: k_mask_fill
    const bool use_qg = large || mask;
    uint32_t prefix = 0, max_qw = 0, pairs = 0;
    for (uint32_t s = 0; s < n; ++s) {
        make_job(d, b.pieces[s], b.h_jobs[s], prefix, use_qg);
        b.h_jobs[s].pair_prefix = pairs;
        prefix += b.h_jobs[s].nblocks;
        pairs += (b.h_jobs[s].nblocks + 1) / 2;
        max_qw = std::max(max_qw, b.h_jobs[s].qg_words);
    }
    cudaStream_t st = d->serial ? d->sync.st : b.st;
    d->h2d_bytes += n * sizeof(SegJob);
    d->d2h_bytes += n * sizeof(DevRecord);
    CU(d, cudaMemcpyAsync(b.d_jobs, b.h_jobs, n * sizeof(SegJob), cudaMemcpyHostToDevice, st));
    CU(d, cudaMemsetAsync(b.d_acc, 0, n * sizeof(SlotAcc), st));
    CU(d, cudaMemsetAsync(b.d_counters, 0, 4 * sizeof(unsigned int), st));
    b.timed = d->timing;
    b.pre = use_qg;
    if (b.timed) CU(d, cudaEventRecord(b.ev_l0, st));
    const uint32_t np = d->iB1 - d->iA0;
    if (np) {
        CU(d, launch_segment_offsets(b.d_jobs, n, d->d_primes, d->d_m64, d->iA0, np, b.d_pmc, st));
        d->launches++;
    }
    if (mask) {
        // writes every mask word of each slot (no memset needed)
        MaskArgs K{};
        K.jobs = b.d_jobs;
        K.nslots = n;
        K.pmc = b.d_pmc;
        K.np = np;
        K.iA0 = d->iA0;
        K.iK0 = d->iK0;
        K.iK1 = d->iB1;
        K.qg = b.d_qg;
        K.qg_stride_words = d->qg_stride;
        CU(d, launch_mask_fill(K, max_qw, st));
        d->launches++;
    } else if (large) {
        CU(d, cudaMemsetAsync(b.d_qg, 0xFF, (size_t)n * d->qg_stride * 4, st));
    }
    if (large) {
        // sparse primes walk the batch once when its slots line up on one
        // wheel axis (consecutive claims); otherwise every large prime takes
        // the per-row path
        LargeBatchTab T{};
        const bool axis = large_batch_tab(b.h_jobs, n, T);
        T.cop = d->ls_cop;
        const uint64_t iLB = axis && d->iLB < d->iL1 ? d->iLB : d->iL1;
        // First-index chain: the row walk's row 0 derives k00 from the last
        // row-walk batch's k00 when this batch's origin lies < 2^32 wheel
        // steps above it (consecutive claims), instead of the 64-bit
        // remainder.  With the chain on, every large-prime launch waits for
        // the previous one (event after its launches), so they run in
        // submission order and a k00 buffer is never rewritten before the
        // next batch has read it.
        const bool rowwalk = axis && d->ls_rows && b.d_k00 != nullptr && d->d_m32 != nullptr;
        if (d->ls_chain && d->last_large != nullptr) CU(d, cudaStreamWaitEvent(st, d->last_large->ev_first, 0));
        const uint32_t* prev = nullptr;
        uint32_t dd = 0;
        const SegJob& j0 = b.h_jobs[0];
        if (rowwalk && d->ls_chain && d->chain_b != nullptr && !j0.qneg && j0.qbase >= d->chain_q0 &&
            (j0.qbase - d->chain_q0) / 6 < (1ull << 32)) {
            prev = d->chain_b->d_k00;
            dd = (uint32_t)((j0.qbase - d->chain_q0) / 6);
        }
        int nl = 0;
        CU(d, launch_large_strike(b.d_jobs, n, d->d_primes, d->d_m64, d->iL0, iLB, b.d_qg, d->qg_stride, b.d_k00,
                                  d->d_m32, rowwalk ? &T : nullptr, prev, dd, &nl, st));
        d->launches += nl;
        if (d->ls_chain) {
            CU(d, cudaEventRecord(b.ev_first, st));
            d->last_large = &b;
            // the per-slot path leaves no usable k00 in this batch
            d->chain_b = rowwalk ? &b : nullptr;
            d->chain_q0 = j0.qbase;
        }
        if (iLB < d->iL1) {
            CU(d, launch_large_batch(b.d_jobs, T, d->d_primes, d->d_m64, iLB, d->iL1, b.d_qg, d->qg_stride, st));
            d->launches++;
        }
    }
    VerifyArgs A{};
    A.jobs = b.d_jobs;
    A.nslots = n;
    A.total_blocks = prefix;
    A.primes = d->d_primes;
    A.n_primes = d->n_primes;
    A.sbound = std::max<uint64_t>(d->sqrt_bound, 47);
    A.iA0 = d->iA0;
    A.iA1 = d->iA1;
    A.iB1 = d->iB1;
    A.iQ1 = d->iQ1;
    A.iH1 = d->iH1;
    A.iW1 = d->iW1;
    A.np = np;
    A.iK0 = mask ? d->iK0 : d->iB1;
    // sieve/check split by the primes the sieve group still visits per block
    // (the row primes; the mask fill takes the rest)
    // (more check warps above 2^44: p_min grows with n, the check with it;
    // C5 window 0.183 s with 12 sieve warps against 0.189 s with 16)
    const uint32_t rows = A.iK0 - d->iA0;
    A.sw = rows > WS_HEAVY_PRIMES && !large ? WS_SW_HEAVY : rows > WS_MASK_PRIMES ? WS_SW_LIGHT : WS_SW_MASK;
    if (d->force_sw) A.sw = d->force_sw;
    A.pmc = b.d_pmc;
    A.wsplit = A.sw == WS_SW_HEAVY ? d->d_wsplit_heavy : A.sw == WS_SW_MASK ? d->d_wsplit_mask : d->d_wsplit;
    A.qg = use_qg ? b.d_qg : nullptr;
    A.qg_stride_words = d->qg_stride;
    A.gpat6 = d->d_pat6;
    A.masks6 = d->d_masks6;
    A.p_small = d->prm.p_small;
    A.inject = d->prm.inject_fail;
    A.block_counter = b.d_counters;
    A.acc = b.d_acc;
    A.list = b.d_list;
    A.list_count = b.d_counters + 1;
    A.list_cap = LIST_CAP;
    A.pmin_out = pmin_out;
    A.total_pairs = pairs;
    A.pair_counter = b.d_counters + 2;
    A.tile_out = tile_out;
    A.tile_fb = tile_fb;
    int grid = std::min<int>(d->sms * d->occ, (int)prefix);
    if (grid < 1) grid = 1;
    if (b.timed) CU(d, cudaEventRecord(b.ev_k0, st));
    if (d->pair) CU(d, launch_verify_pairs(A, grid, st));
    else CU(d, launch_verify_blocks(A, grid, st));
    if (b.timed) CU(d, cudaEventRecord(b.ev_k1, st));
    CU(d, launch_stragglers(b.d_jobs, b.d_list, b.d_counters + 1, LIST_CAP, d->prm.p_small, b.d_res, pmin_out,
                            d->sms, st));
    CU(d, launch_finalize(b.d_jobs, n, b.d_acc, b.d_list, b.d_counters + 1, LIST_CAP, b.d_res, b.d_rec, st));
    if (b.timed) CU(d, cudaEventRecord(b.ev_s1, st));
    d->launches += 3;
    CU(d, cudaMemcpyAsync(b.h_rec, b.d_rec, n * sizeof(DevRecord), cudaMemcpyDeviceToHost, st));
    CU(d, cudaEventRecord(b.ev_done, st));
    b.launched = true;
    return GB_OK;
}

static void rec_merge(gb_seg_record& t, const DevRecord& r) {
    t.evens_checked += r.evens;
    t.unverified_p1 += r.unverified;
    t.phase2_resolved += r.phase2;
    t.pmin_sum += r.pmin_sum;
    t.pmin_hash += r.pmin_hash;
    if (r.max_p != 0 && (r.max_p > t.max_p || (r.max_p == t.max_p && r.max_n < t.max_n))) {
        t.max_p = r.max_p;
        t.max_n = r.max_n;
    }
    uint64_t stored = std::min<uint64_t>(r.n_ce, GB_REC_MAX_CE);
    for (uint64_t i = 0; i < stored; ++i) {
        uint64_t v = r.ce[i];
        uint64_t k = std::min<uint64_t>(t.n_counterexamples, GB_REC_MAX_CE);
        while (k > 0 && t.counterexamples[k - 1] > v) {
            if (k < GB_REC_MAX_CE) t.counterexamples[k] = t.counterexamples[k - 1];
            --k;
        }
        if (k < GB_REC_MAX_CE) t.counterexamples[k] = v;
        t.n_counterexamples++;
    }
    t.n_counterexamples += r.n_ce - stored;
}

static UserSeg* find_seg(gb_dev* d, uint64_t seq) {
    for (auto& u : d->segs)
        if (u.seq == seq) return &u;
    return nullptr;
}

// Run pieces one at a time on the private batch and return the merged record
// (used for the straggler-list overflow fallback and the parity hooks).
static int run_piece_sync(gb_dev* d, uint64_t a, uint64_t b, DevRecord* out, uint64_t* pmin_out) {
    Batch& s = d->sync;
    s.pieces.assign(1, Piece{0, a, b});
    int rc = batch_launch(d, s, pmin_out);
    if (rc) return rc;
    CU(d, cudaEventSynchronize(s.ev_done));
    CU(d, cudaGetLastError());
    s.launched = false;
    *out = s.h_rec[0];
    return GB_OK;
}

static int rerun_split(gb_dev* d, uint64_t a, uint64_t b, gb_seg_record& into) {
    // every straggler entry is one even, so pieces of <= LIST_CAP evens can
    // never overflow the list
    const uint64_t span = 2ull * (LIST_CAP - 16);
    for (uint64_t x = a;; x += span) {
        uint64_t y = (b - x) >= span ? x + span - 2 : b;
        DevRecord r;
        int rc = run_piece_sync(d, x, y, &r, nullptr);
        if (rc) return rc;
        if (r.overflow) GB_FAIL(d, GB_ERR_INTERNAL, "straggler list overflow on a sub-piece");
        rec_merge(into, r);
        if (y == b) break;
    }
    return GB_OK;
}

static int batch_complete(gb_dev* d, int bi) {
    Batch& b = d->batches[bi];
    CU(d, cudaEventSynchronize(b.ev_done));
    CU(d, cudaGetLastError());
    if (b.timed) {
        float ms = 0;
        if (b.pre && cudaEventElapsedTime(&ms, b.ev_l0, b.ev_k0) == cudaSuccess) {
            d->kms[1] += ms;
            d->kl[1] += 1;
        }
        // fused kernel: time from max(own start, previous fused launch's end)
        // to its end, so overlapping launches of consecutive batches are
        // not double counted (their union is the time the kernel runs)
        float t0 = 0, t1 = 0;
        if (cudaEventElapsedTime(&t0, d->t_ref, b.ev_k0) == cudaSuccess &&
            cudaEventElapsedTime(&t1, d->t_ref, b.ev_k1) == cudaSuccess) {
            const double start = std::max<double>(t0, d->last_k1);
            if (t1 > start) d->kms[0] += t1 - start;
            d->last_k1 = std::max<double>(d->last_k1, t1);
            d->kl[0] += 1;
        }
        if (cudaEventElapsedTime(&ms, b.ev_k1, b.ev_s1) == cudaSuccess) {
            d->kms[2] += ms;
            d->kl[2] += 2;
        }
    }
    double t = now_s();
    for (size_t s = 0; s < b.pieces.size(); ++s) {
        UserSeg* u = find_seg(d, b.pieces[s].seq);
        if (!u) GB_FAIL(d, GB_ERR_INTERNAL, "completed piece has no owner");
        const DevRecord& r = b.h_rec[s];
        if (r.overflow) {
            int rc = rerun_split(d, b.pieces[s].a, b.pieces[s].b, u->rec);
            if (rc) return rc;
        } else {
            rec_merge(u->rec, r);
        }
        u->pieces_done++;
        if (u->pieces_done == u->pieces_total) u->rec.elapsed_seconds = t - u->t0;
    }
    b.pieces.clear();
    b.launched = false;
    return GB_OK;
}

static int launch_fill(gb_dev* d) {
    if (d->fill < 0) return GB_OK;
    Batch& b = d->batches[d->fill];
    if (b.pieces.empty()) return GB_OK;
    int rc = batch_launch(d, b, nullptr);
    if (rc) return rc;
    d->inflight.push_back(d->fill);
    d->fill = -1;
    return GB_OK;
}

static int acquire_fill(gb_dev* d) {
    if (d->fill >= 0) return GB_OK;
    for (;;) {
        for (int i = 0; i < NBATCH; ++i) {
            Batch& b = d->batches[i];
            bool busy = b.launched || !b.pieces.empty();
            if (!busy) {
                d->fill = i;
                return GB_OK;
            }
        }
        // all batches in flight: retire the oldest
        if (d->inflight.empty()) GB_FAIL(d, GB_ERR_INTERNAL, "no free batch");
        int bi = d->inflight.front();
        d->inflight.pop_front();
        int rc = batch_complete(d, bi);
        if (rc) return rc;
    }
}

static int check_segment(gb_dev* d, uint64_t a, uint64_t b) {
    // check_job (verifier.cpp:15-20)
    if ((a & 1) || (b & 1)) GB_FAIL(d, GB_ERR_PARAM, "segment bounds must be even");
    if (a < 4 || a > b) GB_FAIL(d, GB_ERR_PARAM, "segment must satisfy 4 <= a <= b");
    // sieve_range_for (verifier.cpp:35-43) and the coverage check of
    // tiled_sieve_segment (sieve.cpp:100-103)
    uint64_t lo = a > d->prm.p_small ? a - d->prm.p_small : 0;
    if (lo < 3) lo = 3;
    if ((lo & 1) == 0) ++lo;
    uint64_t hi = b - 3;
    if (hi < lo) hi = lo;
    uint64_t s = d->sqrt_bound;
    if (s == 0 || s < hi / s)
        GB_FAIL(d, GB_ERR_PARAM, "tiled_sieve_segment: base primes insufficient for segment bound");
    return GB_OK;
}

// --------------------------------------------------------------- K1 build
// Odd primes <= L (L >= 3, L < 2^32 + 2^17) into a new device array: seed
// primes by one CTA, segmented sieve of [3, L] with the tile machinery,
// count / scan / compact.  build_base_primes semantics (sieve.cpp:44-70)
// when L = sqrt_bound.
static int device_odd_primes_upto(gb_dev* d, uint64_t L, uint32_t** d_out, uint64_t* count) {
    cudaStream_t st = d->sync.st;
    *d_out = nullptr;
    *count = 0;
    if (L < 3) {
        CU(d, dmalloc(d->device, d_out, 4));
        return GB_OK;
    }
    uint32_t lim = (uint32_t)std::min<uint64_t>(isqrt_floor(L) + 1, 65536);
    if (lim < 3) lim = 3;
    uint32_t *d_seed = nullptr, *d_nseed = nullptr;
    CU(d, dmalloc(d->device, &d_seed, 8192 * 4));
    CU(d, dmalloc(d->device, &d_nseed, 4));
    CU(d, launch_seed_primes(lim, d_seed, d_nseed, st));
    uint32_t nseed = 0;
    CU(d, cudaMemcpyAsync(&nseed, d_nseed, 4, cudaMemcpyDeviceToHost, st));
    CU(d, cudaStreamSynchronize(st));
    std::vector<uint32_t> hseed(nseed);
    if (nseed) CU(d, cudaMemcpy(hseed.data(), d_seed, nseed * 4, cudaMemcpyDeviceToHost));
    uint32_t sA0 = (uint32_t)(std::lower_bound(hseed.begin(), hseed.end(), FIRST_STRIKE_P) - hseed.begin());
    uint32_t sA1 = (uint32_t)(std::lower_bound(hseed.begin(), hseed.end(), P_WARP_MAX) - hseed.begin());
    const uint64_t n_cells = (L - 3) / 2 + 1;
    const uint64_t n_words = (n_cells + 31) / 32;
    uint32_t* d_bits = nullptr;
    CU(d, dmalloc(d->device, &d_bits, (n_words + 1) * 4));
    int grid = (int)std::min<uint64_t>((n_cells + W - 1) / W, (uint64_t)d->sms * 2);
    CU(d, launch_sieve_interval(3, n_cells, d_seed, sA0, sA1, nseed, d->d_pat, d_bits, grid, st));
    const uint32_t chunk = 4096;
    const uint64_t n_chunks = (n_words + chunk - 1) / chunk;
    uint32_t* d_counts = nullptr;
    uint64_t *d_off = nullptr, *d_total = nullptr;
    CU(d, dmalloc(d->device, &d_counts, n_chunks * 4));
    CU(d, dmalloc(d->device, &d_off, n_chunks * 8));
    CU(d, dmalloc(d->device, &d_total, 8));
    CU(d, launch_count_words(d_bits, n_words, chunk, d_counts, n_chunks, st));
    CU(d, launch_scan(d_counts, n_chunks, d_off, d_total, st));
    uint64_t total = 0;
    CU(d, cudaMemcpyAsync(&total, d_total, 8, cudaMemcpyDeviceToHost, st));
    CU(d, cudaStreamSynchronize(st));
    CU(d, dmalloc(d->device, d_out, std::max<uint64_t>(total, 1) * 4));
    CU(d, launch_compact(d_bits, n_words, chunk, d_off, 3, *d_out, n_chunks, st));
    d->launches += 6;
    CU(d, cudaStreamSynchronize(st));
    dfree(d->device, d_bits);
    dfree(d->device, d_counts);
    dfree(d->device, d_off);
    dfree(d->device, d_total);
    dfree(d->device, d_seed);
    dfree(d->device, d_nseed);
    *count = total;
    return GB_OK;
}

// Mask-fill plan: tile primes >= GB_MASK_P (default M6 + 1: at most one
// multiple per class array of a block window; 0 turns the mask fill off)
// are struck by k_mask_fill once per 3-block range instead of by every
// block's sieve (the reference's sparse-prime hit list, sieve.cpp:109-126,
// in bitmask form).  Off by default (GB_MASK_P=262145 turns it on): measured
// on B200 the fill costs more device time than it takes off the fused kernel
// at 1e12, 1e13 and the C5 window, because it cannot
// share SMs with the persistent kernel while the row visits it replaces run
// beside the check warps.
static int mask_plan(gb_dev* d, const std::vector<uint32_t>& head) {
    d->mk_on = false;
    d->iK0 = d->iB1;
    if (const char* e = getenv("GB_PAIR")) d->pair = atoi(e) != 0;
    if (d->pair && pair_setup() != 0) GB_FAIL(d, GB_ERR_CUDA, "gb_open: cluster kernel attributes");
    if (const char* e = getenv("GB_SW")) {
        const uint32_t v = (uint32_t)atoi(e);
        if (v == WS_SW_LIGHT || v == WS_SW_HEAVY || v == WS_SW_MASK) d->force_sw = v;
    }
    uint64_t pm = 0;
    if (const char* e = getenv("GB_MASK_P")) pm = strtoull(e, nullptr, 0);
    if (pm == 0) return GB_OK;
    pm = std::max<uint64_t>(pm, P_WARP_MAX); // warp-cooperative primes stay on rows
    const uint32_t i = (uint32_t)(std::lower_bound(head.begin(), head.end(), (uint32_t)std::min<uint64_t>(pm, P_TILE_MAX + 1ull)) - head.begin());
    if (i >= d->iB1) return GB_OK; // no tile prime that large
    d->iK0 = std::max(i, d->iA1);
    d->mk_p0 = head[d->iK0];
    d->mk_on = true;
    return GB_OK;
}

static int build_tables(gb_dev* d) {
    CU(d, dmalloc(d->device, &d->d_pat, PAT_WORDS * 4));
    CU(d, dmalloc(d->device, &d->d_pat6, PAT6_WORDS * 4));
    CU(d, dmalloc(d->device, &d->d_masks6, 3 * NWIN6 * 8));
    CU(d, launch_init_tables(d->d_pat, d->d_pat6, d->d_masks6, d->prm.p_small, d->sync.st));
    d->launches++;
    int rc = device_odd_primes_upto(d, d->sqrt_bound, &d->d_primes, &d->n_primes);
    if (rc) return rc;
    const uint64_t total = d->n_primes;
    // index ranges (primes <= P_TILE_MAX are the first pi(2^22) entries)
    uint64_t head = std::min<uint64_t>(total, 300000);
    std::vector<uint32_t> hp(head);
    if (head) CU(d, cudaMemcpy(hp.data(), d->d_primes, head * 4, cudaMemcpyDeviceToHost));
    d->iA0 = (uint32_t)(std::lower_bound(hp.begin(), hp.end(), FIRST_STRIKE_P) - hp.begin());
    d->iA1 = (uint32_t)(std::lower_bound(hp.begin(), hp.end(), P_WARP_MAX) - hp.begin());
    d->iB1 = (uint32_t)(std::upper_bound(hp.begin(), hp.end(), P_TILE_MAX) - hp.begin());
    d->iW1 = std::max(d->iA1, std::min(d->iB1, (uint32_t)(std::lower_bound(hp.begin(), hp.end(), M6) - hp.begin())));
    d->iQ1 = std::max(d->iA1, std::min(d->iW1, (uint32_t)(std::lower_bound(hp.begin(), hp.end(), M6 / 4) - hp.begin())));
    d->iH1 = std::max(d->iQ1, std::min(d->iW1, (uint32_t)(std::lower_bound(hp.begin(), hp.end(), M6 / 2) - hp.begin())));
    d->iL0 = d->iB1;
    d->iL1 = total;
    // warp-cooperative primes [iA0, iA1) to warps, longest first onto the
    // least loaded warp (cost ~ strikes per lane W / 32p + setup); one table
    // per compiled split, the split being chosen per launch (batch_launch)
    for (int h = 0; h < 3; ++h) {
        const int nwarps = h == 0 ? WS_SW_LIGHT : h == 1 ? WS_SW_HEAVY : WS_SW_MASK;
        std::vector<uint16_t> ws(SPLIT_WARPS * 32, 0xFFFF);
        std::vector<double> load(nwarps, 0.0);
        std::vector<int> cnt(nwarps, 0);
        for (uint32_t i = d->iA0; i < d->iA1; ++i) { // ascending p = descending cost
            int best = -1;
            for (int w = 0; w < nwarps; ++w)
                if (cnt[w] < 32 && (best < 0 || load[w] < load[best])) best = w;
            if (best < 0) GB_FAIL(d, GB_ERR_INTERNAL, "too many warp-cooperative primes");
            ws[best * 32 + cnt[best]++] = (uint16_t)(i - d->iA0);
            load[best] += 2.0 * M6 / (32.0 * hp[i]) + 6.0;
        }
        uint16_t*& dst = h == 0 ? d->d_wsplit : h == 1 ? d->d_wsplit_heavy : d->d_wsplit_mask;
        CU(d, dmalloc(d->device, &dst, ws.size() * sizeof(uint16_t)));
        CU(d, cudaMemcpy(dst, ws.data(), ws.size() * sizeof(uint16_t), cudaMemcpyHostToDevice));
    }
    CU(d, dmalloc(d->device, &d->d_m64, std::max<uint64_t>(total, 1) * sizeof(uint64_t)));
    CU(d, launch_prime_magic64(d->d_primes, total, d->d_m64, d->sync.st));
    d->launches++;
    if (d->iL1 > d->iL0 && !(getenv("GB_LS_PRE") && atoi(getenv("GB_LS_PRE")) == 0)) {
        CU(d, dmalloc(d->device, &d->d_m32, (size_t)(d->iL1 - d->iL0) * 4));
        CU(d, launch_large_m32(d->d_m64, d->iL0, d->iL1, d->d_m32, d->sync.st));
        d->launches++;
    }
    // batch-walk threshold (k_large_batch): large primes from GB_LB_T
    // (default 0 = off: measured slower) by a binary search
    // of the device table
    d->iLB = d->iL1;
    if (d->iL1 > d->iL0) {
        uint64_t t = 0;
        if (const char* e = getenv("GB_LB_T")) t = strtoull(e, nullptr, 0);
        if (const char* e = getenv("GB_LS_ROWS")) d->ls_rows = atoi(e) != 0;
        if (const char* e = getenv("GB_LS_COP")) d->ls_cop = (uint32_t)atoi(e);
        if (const char* e = getenv("GB_LS_CHAIN")) d->ls_chain = atoi(e) != 0;
        if (t != 0) {
            uint64_t lo = d->iL0, hi = d->iL1; // first index with p >= t
            while (lo < hi) {
                const uint64_t mid = lo + (hi - lo) / 2;
                uint32_t v = 0;
                CU(d, cudaMemcpy(&v, d->d_primes + mid, 4, cudaMemcpyDeviceToHost));
                if (v < t) lo = mid + 1;
                else hi = mid;
            }
            d->iLB = lo;
        }
    }
    int rc2 = mask_plan(d, hp);
    if (rc2) return rc2;
    CU(d, cudaStreamSynchronize(d->sync.st)); // tables ready before any batch stream
    return GB_OK;
}

static uint64_t pi_upper(uint64_t x) { // Rosser-Schoenfeld style bound, sizing only
    if (x < 17) return 8;
    return (uint64_t)(1.26 * (double)x / std::log((double)x)) + 1;
}

// NVML through dlopen (the driver ships libnvidia-ml.so.1; nothing is
// linked at build time): free/total memory of a CUDA device, matched by PCI
// bus id.  false when NVML is unavailable.
static bool nvml_memory(int device, uint64_t* free_bytes, uint64_t* total_bytes) {
    struct Mem {
        unsigned long long total, free, used;
    };
    using InitFn = int (*)();
    using ByPciFn = int (*)(const char*, void**);
    using MemFn = int (*)(void*, Mem*);
    static std::once_flag once;
    static ByPciFn by_pci = nullptr;
    static MemFn mem = nullptr;
    std::call_once(once, [] {
        void* h = dlopen("libnvidia-ml.so.1", RTLD_NOW | RTLD_LOCAL);
        if (!h) return;
        auto init = reinterpret_cast<InitFn>(dlsym(h, "nvmlInit_v2"));
        by_pci = reinterpret_cast<ByPciFn>(dlsym(h, "nvmlDeviceGetHandleByPciBusId_v2"));
        mem = reinterpret_cast<MemFn>(dlsym(h, "nvmlDeviceGetMemoryInfo"));
        if (!init || !by_pci || !mem || init() != 0) by_pci = nullptr;
    });
    if (!by_pci) return false;
    char bus[32] = {0};
    if (cudaDeviceGetPCIBusId(bus, sizeof(bus), device) != cudaSuccess) return false;
    void* dev = nullptr;
    Mem m{};
    if (by_pci(bus, &dev) != 0 || mem(dev, &m) != 0) return false;
    *free_bytes = m.free;
    *total_bytes = m.total;
    return true;
}

// --------------------------------------------------------------- C-ABI
extern "C" {

const char* gb_version(void) { return "goldbach_b200 1.0 (sm_100a)"; }

int gb_device_count(int* count) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) n = 0;
    *count = n;
    return GB_OK;
}

int gb_open(int device, const gb_params* params, gb_dev** out) {
    *out = nullptr;
    if (!params) GB_FAIL(nullptr, GB_ERR_PARAM, "gb_open: params is NULL");
    if (params->p_small < 3) GB_FAIL(nullptr, GB_ERR_PARAM, "SmallPrimeTable: p_small must be >= 3");
    if (params->cover_limit < 1) GB_FAIL(nullptr, GB_ERR_PARAM, "build_base_primes: cover_limit must be >= 1");
    const double t_enter = now_s();
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
        GB_FAIL(nullptr, GB_ERR_CUDA, "gb_open: no CUDA device available");
    if (device < 0 || device >= n) GB_FAIL(nullptr, GB_ERR_PARAM, "gb_open: device index out of range");
    const double t_count = now_s();
    gb_dev* d = new gb_dev();
    d->device = device;
    d->prm = *params;
    if (d->prm.max_seg_evens == 0) d->prm.max_seg_evens = 200000000ull;
    int rc = GB_OK;
    do {
        if (cudaSetDevice(device) != cudaSuccess) {
            set_err(d, "cudaSetDevice failed");
            rc = GB_ERR_CUDA;
            break;
        }
        // two attributes, not cudaGetDeviceProperties (which queries them all
        // and costs up to ~100 ms per call)
        int major = 0, minor = 0;
        cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
        cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device);
        if (major != 10 || minor != 0) {
            set_err(d, "gb_open: built for sm_100a, device is sm_" + std::to_string(major) + std::to_string(minor));
            rc = GB_ERR_CUDA;
            break;
        }
        cudaDeviceGetAttribute(&d->sms, cudaDevAttrMultiProcessorCount, device);
        const double t_ctx = now_s();
        int occ = 0;
        if (verify_occupancy(&occ) != 0 || occ < 1) {
            set_err(d, "gb_open: fused kernel cannot be resident (shared memory)");
            rc = GB_ERR_RESOURCE;
            break;
        }
        d->occ = occ;
        const double t_open0 = now_s();
        d->sqrt_bound = sqrt_bound_of(params->cover_limit);
        if (cudaStreamCreateWithFlags(&d->sync.st, cudaStreamNonBlocking) != cudaSuccess) {
            set_err(d, "gb_open: cudaStreamCreate failed");
            rc = GB_ERR_CUDA;
            break;
        }
        const double t_open1 = now_s();
        d->max_piece = std::min<uint64_t>(d->prm.max_seg_evens, MAX_PIECE);
        if ((rc = build_tables(d)) != GB_OK) break;
        const double t_open2 = now_s();
        uint64_t blocks = (d->max_piece + E6 - 1) / E6;
        d->qg_stride = 2 * ((blocks * K6 + (M6 - K6) + 31) / 32); // arrays A and B
        if ((rc = batch_alloc(d, d->sync, true)) != GB_OK) break;
        for (int i = 0; i < NBATCH && rc == GB_OK; ++i) rc = batch_alloc(d, d->batches[i], true);
        if (getenv("GB_DEBUG_OPEN") && d->pair) {
            int nc = 0;
            pair_clusters_resident(&nc);
            fprintf(stderr, "gb_open: pair mode, %d two-CTA clusters resident (of %d SMs)\n", nc, d->sms);
        }
        if (getenv("GB_DEBUG_OPEN"))
            fprintf(stderr,
                    "gb_open: driver %.1f ms, context %.1f ms, kernels %.1f ms, setup %.1f ms, tables %.1f ms, "
                    "batches %.1f ms\n",
                    1e3 * (t_count - t_enter), 1e3 * (t_ctx - t_count), 1e3 * (t_open0 - t_ctx),
                    1e3 * (t_open1 - t_open0), 1e3 * (t_open2 - t_open1), 1e3 * (now_s() - t_open2));
    } while (false);
    if (rc != GB_OK) {
        t_err = d->err;
        gb_close(d);
        return rc;
    }
    *out = d;
    return GB_OK;
}

int gb_close(gb_dev* d) {
    if (!d) return GB_OK;
    cudaSetDevice(d->device);
    cudaDeviceSynchronize();
    for (auto& b : d->batches) batch_free(d, b);
    batch_free(d, d->sync);
    if (d->tm0) cudaEventDestroy(d->tm0);
    if (d->tm1) cudaEventDestroy(d->tm1);
    if (d->t_ref) cudaEventDestroy(d->t_ref);
    dfree(d->device, d->d_primes);
    dfree(d->device, d->flush_buf);
    dfree(d->device, d->d_pat);
    dfree(d->device, d->d_pat6);
    dfree(d->device, d->d_masks6);
    dfree(d->device, d->d_wsplit);
    dfree(d->device, d->d_wsplit_heavy);
    dfree(d->device, d->d_wsplit_mask);
    dfree(d->device, d->d_m64);
    dfree(d->device, d->d_m32);
    delete d;
    return GB_OK;
}

const char* gb_last_error(const gb_dev* d) { return d ? d->err.c_str() : t_err.c_str(); }

int gb_set_inject_fail(gb_dev* d, uint64_t inject_fail) {
    if (!d) GB_FAIL(nullptr, GB_ERR_PARAM, "null handle");
    d->prm.inject_fail = inject_fail;
    return GB_OK;
}

int gb_max_inflight(const gb_dev* d, int* depth) {
    (void)d;
    *depth = NBATCH * SLOTS;
    return GB_OK;
}

int gb_submit_segment(gb_dev* d, uint64_t a, uint64_t b, uint64_t tag) {
    if (!d) GB_FAIL(nullptr, GB_ERR_PARAM, "null handle");
    int rc = check_segment(d, a, b);
    if (rc) return rc;
    CU(d, cudaSetDevice(d->device));
    UserSeg u;
    u.seq = d->next_seq++;
    u.a = a;
    u.b = b;
    u.tag = tag;
    u.t0 = now_s();
    u.rec.a = a;
    u.rec.b = b;
    const uint64_t span = 2 * d->max_piece;
    std::vector<Piece> pcs;
    for (uint64_t x = a;; x += span) {
        uint64_t y = (b - x) >= span ? x + span - 2 : b;
        pcs.push_back(Piece{u.seq, x, y});
        if (y == b) break;
    }
    u.pieces_total = (uint32_t)pcs.size();
    d->segs.push_back(u);
    for (const Piece& pc : pcs) {
        if ((rc = acquire_fill(d)) != GB_OK) return rc;
        Batch& fb = d->batches[d->fill];
        fb.pieces.push_back(pc);
        if (fb.pieces.size() == SLOTS)
            if ((rc = launch_fill(d)) != GB_OK) return rc;
    }
    // keep the device busy: launch a partial batch if nothing is running
    if (d->inflight.empty()) rc = launch_fill(d);
    return rc;
}

int gb_wait_segment(gb_dev* d, gb_seg_record* out, uint64_t* tag) {
    if (!d) GB_FAIL(nullptr, GB_ERR_PARAM, "null handle");
    if (d->segs.empty()) GB_FAIL(d, GB_ERR_PARAM, "gb_wait_segment: nothing submitted");
    CU(d, cudaSetDevice(d->device));
    int rc;
    while (d->segs.front().pieces_done < d->segs.front().pieces_total) {
        if (d->inflight.empty()) {
            if (d->fill < 0) GB_FAIL(d, GB_ERR_INTERNAL, "pending segment with no batch");
            if ((rc = launch_fill(d)) != GB_OK) return rc;
            continue;
        }
        // launch the partial batch first so it overlaps the wait
        if (d->fill >= 0 && !d->batches[d->fill].pieces.empty() && (int)d->inflight.size() < NBATCH)
            if ((rc = launch_fill(d)) != GB_OK) return rc;
        int bi = d->inflight.front();
        d->inflight.pop_front();
        if ((rc = batch_complete(d, bi)) != GB_OK) return rc;
    }
    UserSeg u = d->segs.front();
    d->segs.pop_front();
    *out = u.rec;
    if (tag) *tag = u.tag;
    return GB_OK;
}

int gb_verify_segment(gb_dev* d, uint64_t a, uint64_t b, gb_seg_record* out) {
    if (!d) GB_FAIL(nullptr, GB_ERR_PARAM, "null handle");
    if (!d->segs.empty()) GB_FAIL(d, GB_ERR_PARAM, "gb_verify_segment: asynchronous segments pending");
    int rc = gb_submit_segment(d, a, b, 0);
    if (rc) return rc;
    return gb_wait_segment(d, out, nullptr);
}

int gb_base_primes(gb_dev* d, uint64_t* sqrt_bound, uint64_t* count, uint32_t* out, uint64_t cap) {
    if (!d) GB_FAIL(nullptr, GB_ERR_PARAM, "null handle");
    CU(d, cudaSetDevice(d->device));
    if (sqrt_bound) *sqrt_bound = d->sqrt_bound;
    if (count) *count = d->n_primes;
    if (out && cap) {
        uint64_t n = std::min(cap, d->n_primes);
        if (n) CU(d, cudaMemcpy(out, d->d_primes, n * 4, cudaMemcpyDeviceToHost));
    }
    return GB_OK;
}

int gb_sieve_interval(gb_dev* d, uint64_t lo, uint64_t hi, uint64_t* words, uint64_t n_words) {
    if (!d) GB_FAIL(nullptr, GB_ERR_PARAM, "null handle");
    if ((lo & 1) == 0 || (hi & 1) == 0) GB_FAIL(d, GB_ERR_PARAM, "tiled_sieve_segment: bounds must be odd");
    if (lo > hi) GB_FAIL(d, GB_ERR_PARAM, "tiled_sieve_segment: lo must be <= hi");
    uint64_t s = d->sqrt_bound;
    if (s == 0 || s < hi / s)
        GB_FAIL(d, GB_ERR_PARAM, "tiled_sieve_segment: base primes insufficient for segment bound");
    const uint64_t n_cells = ((hi - lo) >> 1) + 1;
    const uint64_t need = (n_cells + 63) / 64;
    if (n_words < need) GB_FAIL(d, GB_ERR_PARAM, "gb_sieve_interval: output too small");
    CU(d, cudaSetDevice(d->device));
    cudaStream_t st = d->sync.st;
    uint32_t* d_bits = nullptr;
    CU(d, dmalloc(d->device, &d_bits, need * 8 + 8));
    CU(d, cudaMemsetAsync(d_bits, 0, need * 8 + 8, st));
    int grid = (int)std::min<uint64_t>((n_cells + W - 1) / W, (uint64_t)d->sms * 2);
    // every base prime (p^2 beyond hi strikes nothing)
    CU(d, launch_sieve_interval(lo, n_cells, d->d_primes, d->iA0, d->iA1, (uint32_t)d->n_primes, d->d_pat, d_bits,
                                grid, st));
    d->launches++;
    CU(d, cudaMemcpyAsync(words, d_bits, need * 8, cudaMemcpyDeviceToHost, st));
    CU(d, cudaStreamSynchronize(st));
    dfree(d->device, d_bits);
    return GB_OK;
}

int gb_phase1_pmin(gb_dev* d, uint64_t a, uint64_t b, uint64_t* out, uint64_t n_out) {
    if (!d) GB_FAIL(nullptr, GB_ERR_PARAM, "null handle");
    int rc = check_segment(d, a, b);
    if (rc) return rc;
    uint64_t n = ((b - a) >> 1) + 1;
    if (n_out < n) GB_FAIL(d, GB_ERR_PARAM, "gb_phase1_pmin: output too small");
    if (n > LIST_CAP - 16) GB_FAIL(d, GB_ERR_PARAM, "gb_phase1_pmin: at most 2^20 evens per call");
    CU(d, cudaSetDevice(d->device));
    uint64_t* d_out = nullptr;
    CU(d, dmalloc(d->device, &d_out, n * 8));
    DevRecord r;
    rc = run_piece_sync(d, a, b, &r, d_out);
    if (rc == GB_OK) CU(d, cudaMemcpy(out, d_out, n * 8, cudaMemcpyDeviceToHost));
    dfree(d->device, d_out);
    return rc;
}

int gb_debug_tile(gb_dev* d, uint64_t a, uint64_t b, uint32_t block, uint32_t* out_words, uint64_t cap_words,
                  uint32_t* words_per_array, int64_t* origin) {
    if (!d || !words_per_array) GB_FAIL(d, GB_ERR_PARAM, "gb_debug_tile: null argument");
    *words_per_array = M6W;
    if (!out_words) return GB_OK; // size query
    if (!origin || cap_words < 2ull * M6W) GB_FAIL(d, GB_ERR_PARAM, "gb_debug_tile: output too small");
    int rc = check_segment(d, a, b);
    if (rc) return rc;
    const uint64_t evens = ((b - a) >> 1) + 1;
    if (evens > d->max_piece) GB_FAIL(d, GB_ERR_PARAM, "gb_debug_tile: segment larger than one piece");
    if (block >= (evens + E6 - 1) / E6) GB_FAIL(d, GB_ERR_PARAM, "gb_debug_tile: no such block");
    CU(d, cudaSetDevice(d->device));
    uint32_t* d_tile = nullptr;
    CU(d, dmalloc(d->device, &d_tile, 2 * M6W * 4));
    Batch& s = d->sync;
    s.pieces.assign(1, Piece{0, a, b});
    rc = batch_launch(d, s, nullptr, d_tile, block);
    if (rc == GB_OK) {
        CU(d, cudaEventSynchronize(s.ev_done));
        CU(d, cudaMemcpy(out_words, d_tile, 2 * M6W * 4, cudaMemcpyDeviceToHost));
        const SegJob& j = s.h_jobs[0];
        const int64_t q = j.qneg ? -(int64_t)j.qbase : (int64_t)j.qbase; // |Q| < 2^63 below the ceiling's reach
        *origin = q + 6 * (int64_t)K6 * block;
    }
    s.launched = false;
    dfree(d->device, d_tile);
    return rc;
}

int gb_is_prime_batch(gb_dev* d, const uint64_t* values, uint8_t* out, uint64_t count) {
    if (!d) GB_FAIL(nullptr, GB_ERR_PARAM, "null handle");
    if (!count) return GB_OK;
    CU(d, cudaSetDevice(d->device));
    cudaStream_t st = d->sync.st;
    uint64_t* dv = nullptr;
    uint8_t* dout = nullptr;
    CU(d, dmalloc(d->device, &dv, count * 8));
    CU(d, dmalloc(d->device, &dout, count));
    CU(d, cudaMemcpyAsync(dv, values, count * 8, cudaMemcpyHostToDevice, st));
    CU(d, launch_is_prime_batch(dv, dout, count, st));
    d->launches++;
    CU(d, cudaMemcpyAsync(out, dout, count, cudaMemcpyDeviceToHost, st));
    CU(d, cudaStreamSynchronize(st));
    dfree(d->device, dv);
    dfree(d->device, dout);
    return GB_OK;
}

int gb_phase2_resolve(gb_dev* d, uint64_t n, uint64_t* p) {
    if (!d) GB_FAIL(nullptr, GB_ERR_PARAM, "null handle");
    if (n < 4 || (n & 1)) GB_FAIL(d, GB_ERR_PARAM, "phase2_resolve: n must be even and >= 4");
    CU(d, cudaSetDevice(d->device));
    cudaStream_t st = d->sync.st;
    uint64_t* dp = nullptr;
    CU(d, dmalloc(d->device, &dp, 8));
    CU(d, launch_phase2_one(n, dp, st));
    d->launches++;
    CU(d, cudaMemcpyAsync(p, dp, 8, cudaMemcpyDeviceToHost, st));
    CU(d, cudaStreamSynchronize(st));
    dfree(d->device, dp);
    return GB_OK;
}

int gb_primes_upto(gb_dev* d, uint64_t limit, uint32_t* out, uint64_t cap, uint64_t* count) {
    if (!d) GB_FAIL(nullptr, GB_ERR_PARAM, "null handle");
    if (limit > 0xFFFFFFFFull) GB_FAIL(d, GB_ERR_RESOURCE, "gb_primes_upto: limit must be < 2^32");
    CU(d, cudaSetDevice(d->device));
    uint32_t* dp = nullptr;
    uint64_t n = 0;
    int rc = device_odd_primes_upto(d, limit, &dp, &n);
    if (rc) return rc;
    if (count) *count = n;
    if (out && cap) {
        uint64_t m = std::min(cap, n);
        if (m) CU(d, cudaMemcpy(out, dp, m * 4, cudaMemcpyDeviceToHost));
    }
    dfree(d->device, dp);
    return GB_OK;
}

uint64_t gb_estimate_device_bytes(uint64_t cover_limit, uint64_t p_small, uint64_t max_seg_evens) {
    (void)p_small;
    if (max_seg_evens == 0) max_seg_evens = 200000000ull;
    const uint64_t s = sqrt_bound_of(cover_limit ? cover_limit : 1);
    const uint64_t np_all = pi_upper(s);
    const uint64_t np_tile = std::min<uint64_t>(np_all, pi_upper(P_TILE_MAX));
    const uint64_t piece = std::min<uint64_t>(max_seg_evens, MAX_PIECE);
    // large-prime bitmask: primes > P_TILE_MAX, or the mask fill (s > M6)
    const uint64_t qg = s > M6 ? SLOTS * 2 * ((((piece + E6 - 1) / E6) * K6 + (M6 - K6) + 31) / 32) * 4 : 0;
    // primes > P_TILE_MAX: per-batch first indices (k_large_first), 4 B each
    const uint64_t np_large = np_all > np_tile ? np_all - np_tile : 0;
    const uint64_t per_batch = SLOTS * np_tile * sizeof(uint4) + qg + np_large * 4 + (uint64_t)LIST_CAP * (sizeof(StragEntry) + sizeof(StragResult)) +
                               SLOTS * (sizeof(SegJob) + sizeof(SlotAcc) + sizeof(DevRecord)) + 64;
    // base primes + their 64-bit magics + the 32-bit magics of the large ones
    // + K1 scratch bitmap (transient) + NBATCH + 1 batches
    return np_all * (4 + 8) + np_large * 4 + (s / 16 + 64) + (uint64_t)(NBATCH + 1) * per_batch;
}

int gb_warm_device(int device) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n)
        GB_FAIL(nullptr, GB_ERR_PARAM, "gb_warm_device: no such device");
    if (cudaSetDevice(device) != cudaSuccess || cudaFree(nullptr) != cudaSuccess)
        GB_FAIL(nullptr, GB_ERR_CUDA, "gb_warm_device: context creation failed");
    return GB_OK;
}

int gb_device_memory(int device, uint64_t* free_bytes, uint64_t* total_bytes) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n)
        GB_FAIL(nullptr, GB_ERR_PARAM, "gb_device_memory: no such device");
    // NVML first: it reads the device's memory without creating a CUDA
    // context, so a resource check over every worker GPU (cli.cpp
    // validate_resources) leaves the contexts to the worker threads, which
    // create them in parallel
    if (nvml_memory(device, free_bytes, total_bytes)) return GB_OK;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    size_t fr = 0, tot = 0;
    cudaError_t e = cudaMemGetInfo(&fr, &tot);
    cudaSetDevice(prev);
    if (e != cudaSuccess) GB_FAIL(nullptr, GB_ERR_CUDA, cudaGetErrorString(e));
    *free_bytes = fr;
    *total_bytes = tot;
    return GB_OK;
}

// Debug counters of a GB_STATS build (tools/variants.sh); GB_ERR_PARAM in
// regular builds.  Not part of the reference interface.
extern "C" int gb_debug_stats(uint64_t* out8, int reset) {
    if (!out8) return GB_ERR_PARAM;
    unsigned long long v[8];
    const int rc = debug_stats(v, reset);
    for (int i = 0; i < 8; ++i) out8[i] = v[i];
    return rc == 0 ? GB_OK : GB_ERR_PARAM;
}

int gb_set_bucket(gb_dev* d, int enabled) {
    if (!d) GB_FAIL(nullptr, GB_ERR_PARAM, "null handle");
    if (!d->segs.empty()) GB_FAIL(d, GB_ERR_PARAM, "gb_set_bucket: segments pending");
    d->mk_off_now = !enabled;
    return GB_OK;
}

int gb_bucket_info(const gb_dev* d, uint64_t* out8) {
    if (!d || !out8) return GB_ERR_PARAM;
    for (int i = 0; i < 8; ++i) out8[i] = 0;
    out8[0] = d->mk_on && !d->mk_off_now;
    out8[1] = d->mk_on ? d->mk_p0 : 0;
    out8[2] = d->mk_on ? d->iB1 - d->iK0 : 0;
    out8[3] = MK_CELLS;
    out8[4] = d->iL1 - d->iL0;
    return GB_OK;
}

int gb_launch_count(const gb_dev* d, uint64_t* launches) {
    if (!d) return GB_ERR_PARAM;
    *launches = d->launches;
    return GB_OK;
}

int gb_kernel_times(gb_dev* d, double* ms4, uint64_t* launches4, int reset) {
    if (!d) return GB_ERR_PARAM;
    for (int i = 0; i < 4; ++i) {
        if (ms4) ms4[i] = d->kms[i];
        if (launches4) launches4[i] = d->kl[i];
        if (reset) {
            d->kms[i] = 0;
            d->kl[i] = 0;
        }
    }
    return GB_OK;
}

int gb_set_timing(gb_dev* d, int enabled) {
    if (!d) return GB_ERR_PARAM;
    if (!d->segs.empty()) GB_FAIL(d, GB_ERR_PARAM, "gb_set_timing: segments pending");
    d->timing = enabled != 0;
    d->serial = enabled == 2;
    if (d->timing) {
        CU(d, cudaSetDevice(d->device));
        if (!d->t_ref) CU(d, cudaEventCreate(&d->t_ref));
        CU(d, cudaDeviceSynchronize());
        CU(d, cudaEventRecord(d->t_ref, d->sync.st));
        CU(d, cudaEventSynchronize(d->t_ref));
        d->last_k1 = 0;
    }
    return GB_OK;
}

int gb_io_bytes(const gb_dev* d, uint64_t* h2d, uint64_t* d2h) {
    if (!d) return GB_ERR_PARAM;
    if (h2d) *h2d = d->h2d_bytes;
    if (d2h) *d2h = d->d2h_bytes;
    return GB_OK;
}

int gb_flush_l2(gb_dev* d) {
    if (!d) GB_FAIL(nullptr, GB_ERR_PARAM, "null handle");
    CU(d, cudaSetDevice(d->device));
    const size_t bytes = 256ull << 20; // > 126 MB L2
    if (!d->flush_buf) CU(d, dmalloc(d->device, &d->flush_buf, bytes));
    CU(d, cudaMemsetAsync(d->flush_buf, d->launches & 0xff, bytes, d->sync.st));
    CU(d, cudaStreamSynchronize(d->sync.st));
    return GB_OK;
}

int gb_synchronize(gb_dev* d) {
    if (!d) GB_FAIL(nullptr, GB_ERR_PARAM, "null handle");
    CU(d, cudaSetDevice(d->device));
    CU(d, cudaDeviceSynchronize());
    return GB_OK;
}

int gb_device_timer(gb_dev* d, int op, double* ms) {
    if (!d) GB_FAIL(nullptr, GB_ERR_PARAM, "null handle");
    CU(d, cudaSetDevice(d->device));
    if (!d->tm0) CU(d, cudaEventCreate(&d->tm0));
    if (!d->tm1) CU(d, cudaEventCreate(&d->tm1));
    // the device is drained on both sides, so the event pair on the private
    // stream brackets every stream's work in between
    CU(d, cudaDeviceSynchronize());
    if (op == 0) {
        CU(d, cudaEventRecord(d->tm0, d->sync.st));
        CU(d, cudaEventSynchronize(d->tm0));
        return GB_OK;
    }
    if (op != 1) GB_FAIL(d, GB_ERR_PARAM, "gb_device_timer: op must be 0 or 1");
    CU(d, cudaEventRecord(d->tm1, d->sync.st));
    CU(d, cudaEventSynchronize(d->tm1));
    float e = 0;
    CU(d, cudaEventElapsedTime(&e, d->tm0, d->tm1));
    if (ms) *ms = e;
    return GB_OK;
}

int gb_smem_peak(gb_dev* d, double* bytes_per_s) {
    if (!d || !bytes_per_s) GB_FAIL(d, GB_ERR_PARAM, "gb_smem_peak: null argument");
    CU(d, cudaSetDevice(d->device));
    cudaStream_t st = d->sync.st;
    uint32_t* sink = nullptr;
    CU(d, dmalloc(d->device, &sink, 4096 * 4));
    cudaEvent_t e0, e1;
    CU(d, cudaEventCreate(&e0));
    CU(d, cudaEventCreate(&e1));
    const int grid = d->sms * 2;
    const uint32_t iters = 1u << 14;
    CU(d, launch_smem_peak(64, sink, grid, st)); // warm-up
    double best = 0;
    for (int rep = 0; rep < 3; ++rep) {
        CU(d, cudaEventRecord(e0, st));
        CU(d, launch_smem_peak(iters, sink, grid, st));
        CU(d, cudaEventRecord(e1, st));
        CU(d, cudaEventSynchronize(e1));
        float ms = 0;
        CU(d, cudaEventElapsedTime(&ms, e0, e1));
        const double bytes = (double)grid * SMEM_PEAK_THREADS * iters * 8 * 16;
        best = std::max(best, bytes / (ms * 1e-3));
    }
    d->launches += 4;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    dfree(d->device, sink);
    *bytes_per_s = best;
    return GB_OK;
}

} // extern "C"
