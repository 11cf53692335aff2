// gb_device.cuh -- device-side constants and arithmetic for the B200
// Goldbach verifier (sm_100a).  See DESIGN.md for the data layout.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace gbk {

// ---------------------------------------------------------------- geometry
// Odd-only tile of the base-prime sieve (K1, k_sieve_interval): W odd cells
// (bits), cell w covers q = q_w + 2w.  JH = 4096 fixes the in-tile Phase 1
// range of the fused kernel: candidates p = 3 + 2j, j < JH (p <= 8193); evens
// whose minimal p is beyond it go to the straggler kernel (K4), which
// continues the same ascending scan from j = JH.
constexpr int JH = 4096;
constexpr int W_LOG2 = 19;
constexpr uint32_t W = 1u << W_LOG2;    // cells per K1 window
constexpr int TILE_WORDS = W / 32;      // u32 words of the window
constexpr int THREADS = 512;            // threads per CTA of k_sieve_interval
// Warp-specialised fused kernel (k_verify_ws): one CTA of WS_THREADS per SM
// (896: 73 registers per thread, fewer spills than 1024 at equal throughput),
// 32 SW sieve threads + the rest checking.  Two splits are compiled; the host
// takes the heavy-sieve one when the block's tile primes exceed
// WS_HEAVY_PRIMES (measured at 896 threads: 12 sieve warps best at 1e12,
// 15-16 at 1e13).
#ifndef GB_WS_SW_LIGHT
#define GB_WS_SW_LIGHT 12
#endif
#ifndef GB_WS_SW_HEAVY
#define GB_WS_SW_HEAVY 16
#endif
#ifndef GB_WS_SW_MASK
#define GB_WS_SW_MASK 10 // sieve warps when the mask fill takes the large primes
#endif
#ifndef GB_WS_THREADS
#define GB_WS_THREADS 896
#endif
constexpr int WS_THREADS = GB_WS_THREADS;
constexpr int WS_SW_LIGHT = GB_WS_SW_LIGHT, WS_SW_HEAVY = GB_WS_SW_HEAVY, WS_SW_MASK = GB_WS_SW_MASK;
// row primes above which the heavy split is taken: beyond every tile (at
// most pi(2^22) rows) since the 1.5 x 2^18 tile (1e13: 12 sieve warps 4.23 s,
// 16 warps 4.35 s; it was 16 below 2^18-cell tiles); GB_SW=16 still selects it
constexpr uint32_t WS_HEAVY_PRIMES = 400000;
// row primes at or below: the 10-sieve-warp split.  Since the word-entry deep
// queue and the 211 / 419 scan bounds, 1e12 (78 K row primes) measured
// 0.336 s with 10 sieve warps against 0.340 s with 12, and 1e13 (216 K)
// 4.10 s against 4.01 s (profiles/r02f_split_retune.txt)
constexpr uint32_t WS_MASK_PRIMES = 120000;
// warps of the group that runs the warp-cooperative strikes (max of the splits)
constexpr int SPLIT_WARPS = WS_SW_HEAVY > WS_SW_LIGHT ? WS_SW_HEAVY : WS_SW_LIGHT;
constexpr uint32_t P_TILE_MAX = 1u << 22; // base primes above: K_large (global strikes)
#ifndef GB_P_WARP_MAX
#define GB_P_WARP_MAX 2048
#endif
constexpr uint32_t P_WARP_MAX = GB_P_WARP_MAX; // primes below: warp-cooperative strikes
constexpr uint32_t FIRST_STRIKE_P = 53;   // primes below are in the presieve patterns
constexpr uint32_t MAX_SEG_EVENS = 1u << 30; // device sub-segment (piece) limit
constexpr uint32_t MAX_SLOTS = 8;             // pieces (slots) per batch launch

// presieve pattern groups (products of small odd primes); pattern bit k is 0
// iff 2k+1 is divisible by a prime of the group.  Stored with wrap-around
// words so four 32-bit windows at any phase are five word loads.
__host__ __device__ constexpr uint32_t pg_p(int g) {
    return g == 0 ? 15015u : g == 1 ? 7429u : g == 2 ? 33263u : 82861u; // 3·5·7·11·13, 17·19·23, 29·31·37, 41·43·47
}
// words per pattern: a 5-word read (presieve_window) at any phase < P fits
__host__ __device__ constexpr uint32_t pat_words(uint32_t P) { return (P + 31) / 32 + 5; }
__host__ __device__ constexpr uint32_t pg_off(int g) {
    return (g > 0 ? pat_words(pg_p(0)) : 0u) + (g > 1 ? pat_words(pg_p(1)) : 0u) +
           (g > 2 ? pat_words(pg_p(2)) : 0u) + (g > 3 ? pat_words(pg_p(3)) : 0u);
}
constexpr uint32_t PAT_WORDS = pg_off(4);
__host__ __device__ constexpr uint32_t pat_prime(int t) {
    return t == 0 ? 3u : t == 1 ? 5u : t == 2 ? 7u : t == 3 ? 11u : t == 4 ? 13u : t == 5 ? 17u
         : t == 6 ? 19u : t == 7 ? 23u : t == 8 ? 29u : t == 9 ? 31u : t == 10 ? 37u
         : t == 11 ? 41u : t == 12 ? 43u : 47u;
}
constexpr int N_PAT_PRIMES = 14;

// ---------------------------------------------------------------- wheel-6
// The fused kernel sieves a wheel-6 tile: array A holds q = Q + 6k
// (q = 1 mod 6), array B holds q = Q + 4 + 6k (q = 5 mod 6), k < M6; Q = 1
// (mod 6) is the block's window origin.  Multiples of 2 and 3 have no cell,
// so a 96 KiB tile spans 6 M6 = 2.36 M integers (odd-only: 1.57 M) and an
// even n meets only the candidates p with n - p = +-1 (mod 6).  Blocks of a
// slot advance by K6 cells (a multiple of 32, so global bitmask words align)
// and hold E6 = 3 K6 evens; consecutive windows overlap by 6 (M6 - K6) > PH6
// integers, the Phase 1 halo.
#ifndef GB_M6
// cells per class array (a multiple of 32).  Larger tiles visit each row prime
// per more cells: 2^18 / 1.25 / 1.375 / 1.5 x 2^18 measured 1e12 0.366 /
// 0.366 / 0.363 / 0.358 s and 1e13 4.68 / 4.52 / 4.46 / 4.35 s (same
// checksums); 1.5 x 2^18 is the largest that fits two tile buffers beside
// 128-entry deep queues (GB_QCAP)
#define GB_M6 393216
#endif
constexpr uint32_t M6 = GB_M6;                // cells per class array
constexpr uint32_t M6W = M6 / 32;             // words per class array
constexpr uint32_t K6 = M6 - 1376;            // block stride in cells (a multiple of 32: 391840 = 32 * 12245)
constexpr uint32_t E6 = 3 * K6;               // evens per block (1175520)
constexpr uint32_t PH6 = 8193;                // in-tile candidates p <= PH6
constexpr int NWIN6 = 22;                     // 64-wide g-windows, g = p div 6 <= 1365
constexpr uint32_t TPAD = 32;                 // zero words before / after each array (misses of branch-free strikes land here)
constexpr uint32_t TILE6_WORDS = 3 * TPAD + 2 * M6W; // [pad][A][pad][B][pad]
static_assert(M6 % 32 == 0 && K6 % 32 == 0 && 6 * (M6 - K6) > PH6 + 5, "wheel-6 block geometry");
// deep-even queue entries: t (class index in the block, < K6 + 32) | ci | window j
constexpr int DQ_CI = K6 + 64 <= (1u << 18) ? 18 : 19;
constexpr int DQ_J = DQ_CI + 2;
static_assert(K6 + 64 <= (1u << DQ_CI) && DQ_J + 5 <= 32, "deep queue entry layout (word entries store t0 + 32)");
static_assert(64 * NWIN6 * 6 >= PH6, "deep windows cover the halo");

// ------------------------------------------------------------- mask fill
// k_mask_fill: one CTA per MK_CELLS cells (3 block strides) of both class
// arrays of a slot's large-prime bitmask, held in shared memory.
constexpr uint32_t MK_CELLS = (M6 <= 262144 ? 3 : 2) * K6; // the most of 3 / 2 strides that fits (a multiple of 32)
constexpr uint32_t MK_WORDS = MK_CELLS / 32;        // per array
constexpr uint32_t MK_THREADS = 512;
constexpr size_t MK_SMEM = 2ull * MK_WORDS * 4;     // 195.6 KB: one CTA per SM
#ifndef GB_MK_INFLIGHT
#define GB_MK_INFLIGHT 4 // rows loaded before their strikes
#endif
constexpr int MK_INFLIGHT = GB_MK_INFLIGHT;
static_assert(MK_CELLS % 32 == 0, "mask ranges align to words");

// wheel-6 presieve groups: pattern bit k is 0 iff a prime of the group
// divides 6k + 1 (3 has no cells)
__host__ __device__ constexpr uint32_t pg6_p(int g) {
    return g == 0 ? 5005u : g == 1 ? 7429u : g == 2 ? 33263u : 82861u; // 5·7·11·13, 17·19·23, 29·31·37, 41·43·47
}
__host__ __device__ constexpr uint32_t pg6_off(int g) {
    return (g > 0 ? pat_words(pg6_p(0)) : 0u) + (g > 1 ? pat_words(pg6_p(1)) : 0u) +
           (g > 2 ? pat_words(pg6_p(2)) : 0u) + (g > 3 ? pat_words(pg6_p(3)) : 0u);
}
constexpr uint32_t PAT6_WORDS = pg6_off(4);
// 6^-1 mod x for x coprime to 6
__host__ __device__ constexpr uint32_t inv6_mod(uint32_t x) {
    return x % 6 == 1 ? (uint32_t)((5ull * x + 1) / 6) : (uint32_t)((x + 1) / 6);
}

// straggler list entry flags
constexpr uint32_t F_NEED_P1 = 1u;      // continue Phase 1 from j_next
constexpr uint32_t F_P1_FAIL = 2u;      // Phase 1 exhausted: unverified
constexpr uint32_t F_INJECT = 4u;       // n == inject_fail
constexpr uint32_t F_OBSERVED = 8u;     // Phase 1 p already observed in-tile

struct StragEntry {
    uint32_t slot;
    uint32_t i_seg;   // even index within the segment
    uint32_t j_next;  // next candidate index (p = 3 + 2j)
    uint32_t flags;
};

struct StragResult {
    uint64_t p1;      // Phase 1 minimal p found by K4 (0 = none)
    uint64_t p2;      // Phase 2 minimal p (0 = none / not run)
};

// Device-side per-segment job (one per batch slot).  Block b of the slot
// has window origin Q_b = Q + 6 K6 b and evens a + 2 E6 b ...; Q = the
// largest q = 1 (mod 6) with q <= a - PH6, possibly negative near the start
// of the number line (then qneg = 1 and qbase = -Q).
struct SegJob {
    uint64_t a, b;          // evens [a, b]
    uint64_t qbase;         // |Q|
    uint32_t evens;         // (b - a)/2 + 1  (<= MAX_SEG_EVENS)
    uint32_t nblocks;       // ceil(evens / E6)
    uint32_t block_prefix;  // flat index of this slot's first block
    uint32_t qneg;          // Q = -qbase
    uint32_t qg_words;      // words per class array of the large-prime bitmask (0 = none)
    uint32_t delta;         // a - Q (in [PH6, PH6 + 5])
    uint32_t qmod[4];       // Q mod pg6_p(g) (non-negative)
    uint32_t pair_prefix;   // flat index of this slot's first block pair (k_verify_pair)
    uint32_t pad_;
};

// Per-slot accumulator written by the kernels.
struct SlotAcc {
    unsigned long long sum;     // Σ p (tile-certified)
    unsigned long long hash;    // Σ p·(n>>1)
    unsigned long long key;     // max (p << 32 | ~i) over tile-certified evens
    unsigned long long pad;
};

// ---------------------------------------------------------------- helpers
__host__ __device__ __forceinline__ uint64_t first_cell_u64(uint64_t q_w, uint64_t p) {
    // Cell (relative to odd q_w) of the first odd multiple of p that is
    // >= max(p^2, q_w): first_tile_index semantics (sieve.cpp:72-89) without
    // ever forming q_w + d, so it cannot wrap near 2^64.
    uint64_t pp = p * p; // p < 2^32
    if (pp >= q_w) return (pp - q_w) >> 1;
    uint64_t r = q_w % p;
    uint64_t d = r ? p - r : 0;
    if (d & 1) d += p;
    return d >> 1;
}

#ifdef __CUDACC__
// first_cell_u64 with the 64-bit remainder through the prime's magic
// m64 = floor(2^64 / p): the quotient estimate umulhi(q_w, m64) is exact or
// one low, so one correction (instead of a software 64-bit division).
__device__ __forceinline__ uint64_t first_cell_magic(uint64_t q_w, uint64_t p, uint64_t m64) {
    const uint64_t pp = p * p;
    if (pp >= q_w) return (pp - q_w) >> 1;
    uint64_t r = q_w - __umul64hi(q_w, m64) * p;
    if (r >= p) r -= p;
    uint64_t d = r ? p - r : 0;
    if (d & 1) d += p;
    return d >> 1;
}
#endif

// ------------------------------------------------ Miller-Rabin (K4)
// Deterministic for n < 2^64 with witnesses {2..37}: the same decision
// procedure as is_prime_u64 (primality.cpp:32-52), with Montgomery
// multiplication in place of the 128-bit '%'.
struct Mont {
    uint64_t n, ninv, r1; // r1 = 2^64 mod n (Montgomery 1)
};

__device__ __forceinline__ uint64_t mont_mul(uint64_t a, uint64_t b, const Mont& m) {
    uint64_t lo = a * b, hi = __umul64hi(a, b);
    uint64_t q = lo * m.ninv;
    uint64_t mhi = __umul64hi(q, m.n);
    // lo + q*n == 0 mod 2^64; carry out of the low half is (lo != 0)
    uint64_t c = lo != 0;
    uint64_t r = hi + mhi;
    bool ov = r < hi;
    uint64_t r2 = r + c;
    ov |= r2 < r;
    if (ov || r2 >= m.n) r2 -= m.n;
    return r2;
}

__device__ __forceinline__ Mont mont_init(uint64_t n) {
    Mont m;
    m.n = n;
    uint64_t x = n; // n*x == 1 mod 2^3 for odd n
    for (int i = 0; i < 5; ++i) x *= 2 - n * x;
    m.ninv = 0 - x;
    m.r1 = (0 - n) % n;
    return m;
}

__device__ __forceinline__ uint64_t addmod(uint64_t a, uint64_t b, uint64_t n) {
    uint64_t s = a + b;
    if (s < a || s >= n) s -= n;
    return s;
}

__device__ __forceinline__ bool mr_witness(uint64_t a, uint64_t d, int s, const Mont& m) {
    // aR mod n = a * r1 mod n by repeated addition (a <= 37)
    uint64_t aR = 0;
    for (uint64_t k = 0; k < a; ++k) aR = addmod(aR, m.r1, m.n);
    uint64_t x = m.r1;
    uint64_t base = aR;
    uint64_t e = d;
    while (e) {
        if (e & 1) x = mont_mul(x, base, m);
        base = mont_mul(base, base, m);
        e >>= 1;
    }
    uint64_t one = m.r1, minus1 = m.n - m.r1;
    if (x == one || x == minus1) return true;
    for (int r = 1; r < s; ++r) {
        x = mont_mul(x, x, m);
        if (x == minus1) return true;
    }
    return false;
}

__device__ __forceinline__ bool is_prime_u64_dev(uint64_t n) {
    const uint32_t w[12] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    if (n < 41) {
        for (int i = 0; i < 12; ++i)
            if (n == w[i]) return true;
        return false;
    }
    for (int i = 0; i < 12; ++i)
        if (n % w[i] == 0) return false;
    uint64_t d = n - 1;
    int s = 0;
    while ((d & 1) == 0) {
        d >>= 1;
        ++s;
    }
    Mont m = mont_init(n);
    for (int i = 0; i < 12; ++i)
        if (!mr_witness(w[i], d, s, m)) return false;
    return true;
}

} // namespace gbk
