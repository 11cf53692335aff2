// gb_kernels.cu -- sm_100a kernels of the B200 Goldbach verifier.
//
//   K1  k_seed_primes / k_sieve_interval / k_count_words / k_scan /
//       k_compact          base primes <= sqrt_bound on device
//                          (build_base_primes, sieve.cpp:44-70)
//   K2+K3 k_verify_blocks  fused segmented sieve (shared-memory bit tile,
//                          presieve patterns + atomicAnd strikes) and the
//                          Goldbach minimal-p check over the same tile
//                          (tiled_sieve_segment sieve.cpp:91-156 +
//                          phase1_verify verifier.cpp:45-104)
//       k_segment_offsets  per-segment first-multiple cells of tile primes
//       k_large_strike     primes > P_TILE_MAX struck into an L2-resident
//                          segment bitmask (global REDs), ANDed by K2
//   K4  k_stragglers       Phase 1 continuation past the in-tile halo and
//                          Phase 2 (phase2_resolve, verifier.cpp:129-165)
//                          with device Miller-Rabin
//       k_finalize         per-segment record (verify_segment's report,
//                          verifier.cpp:167-206, + checksum)
#include "gb_kernels.h"
#include "gb_bitslice.cuh"

#include <algorithm>
#include <cstdio>


namespace gbk {

#ifdef GB_STATS
// debug counters (variant builds only): 0 generic evens, 1 in-place deep
// evens (queue overflow), 2 queued deep evens, 3 deep rounds, 4 stragglers,
// 5 fast blocks, 6 generic blocks, 7 large-prime REDs outside their slot's
// bitmask (GB_LS_BOUNDS builds: counted and dropped; must stay 0)
__device__ unsigned long long g_stats[8];
#define GB_STAT(i, v) atomicAdd(&g_stats[i], (unsigned long long)(v))
#else
#define GB_STAT(i, v) ((void)0)
#endif

// single-strike rows loaded before their strikes, by sieve-group size.  Since
// the IMAD-addressed strikes (17 instructions per row) 12 rows per thread
// measured best for the 12-warp split (1e13 3.88 s; 8 / 10 / 16 / 20: 3.89 /
// 3.89 / 3.93 / 3.93 s); 1e12 (10 sieve warps, the HEAVY value) is flat over
// 8 / 12 / 16 (profiles/r02f_rows_inflight_ab.txt)
#ifndef GB_RUN_INFLIGHT
#define GB_RUN_INFLIGHT 4 // run-prime rows loaded before their strikes
#endif
#ifndef GB_SS_INFLIGHT_LIGHT
#define GB_SS_INFLIGHT_LIGHT 12
#endif
#ifndef GB_SS_INFLIGHT_HEAVY
#define GB_SS_INFLIGHT_HEAVY 12
#endif
#ifndef GB_RED_ADDR32
#define GB_RED_ADDR32 1 // warp-cooperative strikes as REDs on 32-bit shared addresses
#endif
#ifndef GB_CLASS_TEMPLATE
#define GB_CLASS_TEMPLATE 1 // per-class scan + sums instantiated with immediate constants
#endif
#ifndef GB_PRED_STRIKE
#define GB_PRED_STRIKE 1 // single-strike primes: predicated RED instead of a branch
#endif

// ============================================================ table init
// Presieve patterns (odd-only for K1, wheel-6 for the fused kernel) and the
// wheel-6 deep masks: masks6[c * NWIN6 + j] bit 63 - m set iff p = 6 g + off_c (g = 64 j
// + m; off = +1, -1, +5 for c = 0, 1, 2) is prime, 5 <= p <= min(p_small, PH6).
__device__ bool small_prime(uint32_t p) {
    if (p < 2) return false;
    for (uint32_t d = 2; d * d <= p; ++d)
        if (p % d == 0) return false;
    return true;
}

__global__ void k_init_tables(uint32_t* pat, uint32_t* pat6, uint64_t* masks6, uint64_t p_small) {
    const uint32_t gp[4][3] = {{3, 5, 7}, {17, 19, 23}, {29, 31, 37}, {41, 43, 47}};
    const uint32_t gp1x[2] = {11, 13};
    uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t nthr = gridDim.x * blockDim.x;
    for (int g = 0; g < 4; ++g) {
        uint32_t P = pg_p(g);
        uint32_t nw = pg_off(g + 1) - pg_off(g);
        for (uint32_t w = tid; w < nw; w += nthr) {
            uint32_t v = 0;
            for (int bit = 0; bit < 32; ++bit) {
                uint32_t k = (w * 32 + bit) % P;
                uint32_t q = 2 * k + 1; // odd value represented (mod 2P)
                bool comp = false;
                for (int t = 0; t < 3; ++t) comp |= (q % gp[g][t]) == 0;
                if (g == 0) comp |= (q % gp1x[0]) == 0 || (q % gp1x[1]) == 0;
                if (!comp) v |= 1u << bit;
            }
            pat[pg_off(g) + w] = v;
        }
        // wheel-6: bit k <-> 6k + 1 (mod P); group 0 is 5·7·11·13
        const uint32_t P6 = pg6_p(g);
        const uint32_t nw6 = pg6_off(g + 1) - pg6_off(g);
        for (uint32_t w = tid; w < nw6; w += nthr) {
            uint32_t v = 0;
            for (int bit = 0; bit < 32; ++bit) {
                const uint32_t val = 6u * ((w * 32 + bit) % P6) + 1; // < 6 * 82861 + 1
                bool comp = false;
                if (g == 0) comp = val % 5 == 0 || val % 7 == 0 || val % 11 == 0 || val % 13 == 0;
                else for (int t = 0; t < 3; ++t) comp |= (val % gp[g][t]) == 0;
                if (!comp) v |= 1u << bit;
            }
            pat6[pg6_off(g) + w] = v;
        }
    }
    // one warp per mask word, one candidate per lane and half
    const uint64_t pmax = p_small < PH6 ? p_small : PH6;
    const uint32_t lane = threadIdx.x & 31;
    for (uint32_t e = tid >> 5; e < 3u * NWIN6; e += nthr >> 5) {
        const uint32_t cls = e / NWIN6, j = e % NWIN6;
        const int off = cls == 0 ? 1 : cls == 1 ? -1 : 5;
        uint32_t half[2];
        for (int h = 0; h < 2; ++h) {
            const int64_t p = 6 * (int64_t)(64 * j + 32 * h + lane) + off;
            half[h] = __ballot_sync(0xffffffffu, p >= 5 && (uint64_t)p <= pmax && small_prime((uint32_t)p));
        }
        // bit 63 - jm <-> candidate jm
        if (lane == 0) masks6[e] = ((uint64_t)__brev(half[0]) << 32) | __brev(half[1]);
    }
}

// ============================================================ K1
// Odd primes <= lim (lim <= 65536) by one CTA: seeds for the table sieve.
__global__ void k_seed_primes(uint32_t lim, uint32_t* out, uint32_t* count) {
    __shared__ uint32_t bits[65536 / 64 + 1]; // bit i <-> 2i+1
    const uint32_t nb = lim / 2 + 1;
    for (uint32_t i = threadIdx.x; i < (nb + 31) / 32; i += blockDim.x) bits[i] = ~0u;
    __syncthreads();
    for (uint32_t p = 3 + 2 * threadIdx.x; p * p <= lim; p += 2 * blockDim.x) {
        for (uint32_t m = p * p; m <= lim; m += 2 * p) atomicAnd(&bits[m >> 6], ~(1u << ((m >> 1) & 31)));
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t c = 0;
        for (uint32_t v = 3; v <= lim; v += 2)
            if ((bits[v >> 6] >> ((v >> 1) & 31)) & 1) out[c++] = v;
        *count = c;
    }
}

// ------------------------------------------------------------ tile sieve
// Presieve (patterns), fix-ups and strikes of one W-cell window in shared
// memory.  OffsetFn(i, p) returns the window cell of the first odd multiple
// of p >= max(p^2, q_w), or >= W when p does not strike the window.

__device__ __forceinline__ void presieve_window(uint32_t* tile, const uint32_t* pat, uint64_t q_w, uint32_t tid,
                                                uint32_t nthr) {
    // Each thread builds 4 consecutive tile words per step (one 16-B store):
    // per pattern group 5 loads and 4 funnel shifts at one bit phase o,
    // o = pattern bit of the first cell, advanced by 128 * blockDim mod P.
    uint32_t o[4], step[4];
    const uint64_t k0 = (q_w - 1) >> 1;
#pragma unroll
    for (int g = 0; g < 4; ++g) {
        const uint32_t P = pg_p(g);
        const uint32_t ph = (uint32_t)(k0 % P);
        o[g] = (uint32_t)((ph + 128ull * tid) % P);
        step[g] = (128u * nthr) % P;
    }
    for (uint32_t wd = 4 * tid; wd < (uint32_t)TILE_WORDS; wd += 4 * nthr) {
        uint4 v = make_uint4(~0u, ~0u, ~0u, ~0u);
#pragma unroll
        for (int g = 0; g < 4; ++g) {
            const uint32_t* pg = pat + pg_off(g) + (o[g] >> 5);
            const uint32_t sh = o[g]; // funnel shifts use sh mod 32
            const uint32_t w0 = pg[0], w1 = pg[1], w2 = pg[2], w3 = pg[3], w4 = pg[4];
            v.x &= __funnelshift_r(w0, w1, sh);
            v.y &= __funnelshift_r(w1, w2, sh);
            v.z &= __funnelshift_r(w2, w3, sh);
            v.w &= __funnelshift_r(w3, w4, sh);
            const uint32_t on = o[g] + step[g];
            o[g] = min(on, on - pg_p(g)); // on < 2P
        }
        *reinterpret_cast<uint4*>(tile + wd) = v;
    }
}

// After presieve: restore the pattern primes themselves and clear q = 1.
__device__ __forceinline__ void presieve_fixup(uint32_t* tile, uint64_t q_w, uint32_t tid) {
    if (tid == 0 && q_w <= 47) {
        if (q_w == 1) atomicAnd(&tile[0], ~1u);
#pragma unroll
        for (int t = 0; t < 14; ++t) {
            uint64_t p = pat_prime(t);
            if (p >= q_w) {
                uint64_t c = (p - q_w) >> 1;
                if (c < W) atomicOr(&tile[c >> 5], 1u << (c & 31));
            }
        }
    }
}

__device__ __forceinline__ void strike(uint32_t* tile, uint32_t c) {
    // ~(1 << (c & 31)) as one rotate of 0xFFFFFFFE
    atomicAnd(&tile[c >> 5], __funnelshift_l(0xFFFFFFFEu, 0xFFFFFFFEu, c));
}

// strikes c, c + step, ... < W (two per trip)
__device__ __forceinline__ void strike_run(uint32_t* tile, uint32_t c, uint32_t step) {
    while (c + step < W) {
        strike(tile, c);
        strike(tile, c + step);
        c += 2 * step;
    }
    if (c < W) strike(tile, c);
}

// warp-cooperative strikes (p < P_WARP_MAX) then thread-per-prime strikes.
// OffsetFn::small(i, p) / OffsetFn::large(i, p): window cell of the first
// odd multiple of p >= max(p^2, q_w), or >= W when p misses the window.
template <class OffsetFn>
__device__ __forceinline__ void strike_primes(uint32_t* tile, const uint32_t* __restrict__ primes,
                                              uint32_t iA0, uint32_t iA1, uint32_t iB1,
                                              const OffsetFn& off_of) {
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t nwarps = blockDim.x >> 5;
    for (uint32_t i = iA0 + warp; i < iA1; i += nwarps) {
        uint32_t p = primes[i];
        uint32_t off = off_of.small(i, p);
        if (off >= W) continue;
        strike_run(tile, off + lane * p, 32 * p);
    }
    for (uint32_t i = iA1 + threadIdx.x; i < iB1; i += blockDim.x) {
        uint32_t p = __ldg(primes + i);
        strike_run(tile, off_of.large(i, p), p);
    }
}

// Generic window offset from a 64-bit window start (K1 / interval sieve).
struct DirectOffset {
    uint64_t q_w;
    __device__ __forceinline__ uint32_t small(uint32_t, uint32_t p) const {
        uint64_t c = first_cell_u64(q_w, p);
        return c < W ? (uint32_t)c : W;
    }
    __device__ __forceinline__ uint32_t large(uint32_t i, uint32_t p) const { return small(i, p); }
};

// Sieve-only kernel: bits of odd [lo, hi] into out (cell i <-> lo + 2i),
// cells past hi cleared.  primes: odd primes covering hi (p^2 > hi ignored).
__global__ void __launch_bounds__(THREADS) k_sieve_interval(uint64_t lo, uint64_t n_cells,
                                                            const uint32_t* __restrict__ primes,
                                                            uint32_t iA0, uint32_t iA1, uint32_t iB1,
                                                            const uint32_t* __restrict__ gpat,
                                                            uint32_t* __restrict__ out) {
    extern __shared__ __align__(16) uint32_t smem[];
    uint32_t* tile = smem;                       // TILE_WORDS + 1
    uint32_t* pat = smem + TILE_WORDS + 1;       // PAT_WORDS
    for (uint32_t i = threadIdx.x; i < PAT_WORDS; i += blockDim.x) pat[i] = gpat[i];
    __syncthreads();
    const uint64_t nblk = (n_cells + W - 1) / W;
    for (uint64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
        const uint64_t q_w = lo + 2 * blk * (uint64_t)W;
        presieve_window(tile, pat, q_w, threadIdx.x, blockDim.x);
        __syncthreads();
        presieve_fixup(tile, q_w, threadIdx.x);
        strike_primes(tile, primes, iA0, iA1, iB1, DirectOffset{q_w});
        __syncthreads();
        const uint64_t base_word = blk * (W / 32);
        const uint64_t total_words = (n_cells + 31) / 32;
        for (uint32_t wd = threadIdx.x; wd < (uint32_t)TILE_WORDS; wd += blockDim.x) {
            uint64_t gw = base_word + wd;
            if (gw >= total_words) break;
            uint32_t v = tile[wd];
            uint64_t cell0 = gw * 32;
            if (cell0 + 32 > n_cells) v &= (1u << (n_cells - cell0)) - 1; // n_cells - cell0 < 32
            out[gw] = v;
        }
        __syncthreads();
    }
}

__global__ void k_count_words(const uint32_t* __restrict__ bits, uint64_t n_words, uint32_t chunk,
                              uint32_t* __restrict__ counts) {
    // counts[c] = popcount of words [c*chunk, (c+1)*chunk)
    uint64_t c = blockIdx.x;
    uint64_t w0 = c * chunk, w1 = min((uint64_t)(c + 1) * chunk, n_words);
    uint32_t s = 0;
    for (uint64_t w = w0 + threadIdx.x; w < w1; w += blockDim.x) s += __popc(bits[w]);
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    __shared__ uint32_t red[32];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (uint32_t i = 0; i < blockDim.x / 32; ++i) t += red[i];
        counts[c] = t;
    }
}

// exclusive scan of n counts (single CTA, serial chunks) -> offsets; total
__global__ void k_scan(const uint32_t* counts, uint64_t n, uint64_t* offsets, uint64_t* total) {
    __shared__ uint64_t part[1024];
    uint64_t per = (n + blockDim.x - 1) / blockDim.x;
    uint64_t i0 = threadIdx.x * per, i1 = min(i0 + per, n);
    uint64_t s = 0;
    for (uint64_t i = i0; i < i1; ++i) s += counts[i];
    part[threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t run = 0;
        for (uint32_t t = 0; t < blockDim.x; ++t) {
            uint64_t v = part[t];
            part[t] = run;
            run += v;
        }
        *total = run;
    }
    __syncthreads();
    uint64_t run = part[threadIdx.x];
    for (uint64_t i = i0; i < i1; ++i) {
        offsets[i] = run;
        run += counts[i];
    }
}

// primes[offset..] = lo + 2*(bit index) for each set bit, in order.
__global__ void k_compact(const uint32_t* __restrict__ bits, uint64_t n_words, uint32_t chunk,
                          const uint64_t* __restrict__ offsets, uint64_t lo, uint32_t* __restrict__ primes) {
    uint64_t c = blockIdx.x;
    uint64_t w0 = c * chunk, w1 = min((uint64_t)(c + 1) * chunk, n_words);
    __shared__ uint32_t wsum[33];
    uint64_t base = offsets[c];
    // process the chunk in rounds of blockDim.x words, preserving order
    for (uint64_t r0 = w0; r0 < w1; r0 += blockDim.x) {
        uint64_t w = r0 + threadIdx.x;
        uint32_t v = w < w1 ? bits[w] : 0;
        uint32_t cnt = __popc(v);
        // block exclusive scan of cnt
        uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        uint32_t x = cnt;
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= (uint32_t)o) x += y;
        }
        if (lane == 31) wsum[warp] = x;
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t run = 0;
            for (uint32_t k = 0; k < blockDim.x / 32; ++k) {
                uint32_t t = wsum[k];
                wsum[k] = run;
                run += t;
            }
            wsum[32] = run;
        }
        __syncthreads();
        uint64_t pos = base + wsum[warp] + (x - cnt);
        while (v) {
            uint32_t bit = __ffs(v) - 1;
            v &= v - 1;
            primes[pos++] = (uint32_t)(lo + 2 * (w * 32 + bit));
        }
        base += wsum[32];
        __syncthreads();
    }
}

// ============================================================ segment setup
// x mod p through the prime's 64-bit magic (quotient estimate exact or one low)
__device__ __forceinline__ uint64_t mod_magic(uint64_t x, uint64_t p, uint64_t m64) {
    const uint64_t r = x - __umul64hi(x, m64) * p;
    return r >= p ? r - p : r;
}

// 4 6^-1 mod p (array B's first index is A's minus this), without a division
__device__ __forceinline__ uint32_t b_shift6(uint32_t p) {
    uint64_t c = 4ull * inv6_mod(p); // < 4p
    while (c >= p) c -= p;
    return (uint32_t)c;
}

// First index k >= 0 of array A (q = Q + 6k) with p | q: (-Q) 6^-1 mod p.
__device__ __forceinline__ uint32_t first_a6(const SegJob& J, uint32_t p, uint64_t m64) {
    uint64_t r = mod_magic(J.qbase, p, m64); // |Q| mod p
    if (!J.qneg) r = r ? p - r : 0;          // (-Q) mod p
    return (uint32_t)mod_magic(r * inv6_mod(p), p, m64);
}

// pmc[s*np + i] = {p, floor(2^32/p), k0 + p ceil(2^29/p), p - (4 6^-1 mod p)}
// of tile prime i (index iA0 + i), k0 = first_a6 at the slot's window origin;
// array B's first index is k0 - 4 6^-1 (mod p) (block_off6).  Strikes start at the first multiple in
// the window, not at p^2: multiples below p^2 are composite anyway, and q = p
// itself is restored by the low-window fix-up (fixup_low6).
__global__ void k_segment_offsets(const SegJob* __restrict__ jobs, uint32_t nslots,
                                  const uint32_t* __restrict__ primes, const uint64_t* __restrict__ m64,
                                  uint32_t iA0, uint32_t np, uint4* __restrict__ pmc) {
    // grid: x over primes, y = slot (no 64-bit index division)
    const uint32_t s = blockIdx.y;
    const SegJob& J = jobs[s];
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < np; i += gridDim.x * blockDim.x) {
        const uint32_t p = primes[iA0 + i];
        const uint32_t k0 = first_a6(J, p, m64[iA0 + i]);
        const uint32_t zk = k0 + p * (((1u << 29) + p - 1) / p); // < 2^29 + 2p
        pmc[(size_t)s * np + i] = make_uint4(p, (uint32_t)((1ull << 32) / p), zk, p - b_shift6(p));
    }
}

// Primes above P_TILE_MAX: strike each slot's global wheel-6 bitmask (array A
// then array B, qg_words words each, cells relative to the slot's origin)
// with RED.AND; the fused kernel ANDs the words into its tiles.  One thread
// per prime for every slot of the batch: p and its magic are loaded once, the
// full first-multiple computation runs for slot 0 only, and a slot whose
// origin lies d < 2^32 wheel steps above slot 0's (consecutive pool claims)
// gets its first index as k0 - d mod p with 32-bit arithmetic.
constexpr uint32_t LS_MAX_SLOTS = 16;
#ifndef GB_LS_GROUP
#define GB_LS_GROUP 2
#endif
// slots per grid row: the rows run in order, so the REDs of one row hit
// LS_GROUP slot bitmasks (16.7 MB each at 2e8-even segments) that stay in L2
constexpr uint32_t LS_GROUP = GB_LS_GROUP;

// 4 6^-1 mod p = 2 3^-1 mod p in closed form (p > 3 prime): (p + 2)/3 for
// p = 1 (mod 3), (2p + 2)/3 for p = 2 (mod 3).  No loop, no 64-bit product.
__device__ __forceinline__ uint32_t b_shift6_cf(uint32_t p) {
    const uint32_t q3 = p / 3, r3 = p - 3 * q3;
    return r3 == 1 ? q3 + 1 : 2 * q3 + 2;
}

// Once per batch: k00[i] = first index of array A at slot 0's window origin
// for every prime above P_TILE_MAX (the 64-bit remainder), so that the
// k_large_strike grid rows (one per LS_GROUP slots) derive their slots'
// first indices with 32-bit arithmetic instead of each recomputing it.
__global__ void __launch_bounds__(256) k_large_first(const SegJob* __restrict__ jobs,
                                                     const uint32_t* __restrict__ primes,
                                                     const uint64_t* __restrict__ m64, uint64_t iL0, uint64_t iL1,
                                                     uint32_t* __restrict__ k00) {
    const SegJob J = jobs[0];
    for (uint64_t i = iL0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < iL1;
         i += (uint64_t)gridDim.x * blockDim.x)
        k00[i - iL0] = first_a6(J, primes[i], m64[i]);
}

// m32[i] = floor(2^32 / p_i) = m64[i] >> 32, once per open
__global__ void k_large_m32(const uint64_t* __restrict__ m64, uint64_t iL0, uint64_t iL1, uint32_t* __restrict__ m32) {
    for (uint64_t i = iL0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < iL1;
         i += (uint64_t)gridDim.x * blockDim.x)
        m32[i - iL0] = (uint32_t)(m64[i] >> 32);
}

__global__ void __launch_bounds__(256) k_large_strike(const SegJob* __restrict__ jobs, uint32_t nslots,
                                                      const uint32_t* __restrict__ primes,
                                                      const uint64_t* __restrict__ m64, uint64_t iL0, uint64_t iL1,
                                                      uint32_t* __restrict__ qg, uint64_t qg_stride_words,
                                                      const uint32_t* __restrict__ k00s,
                                                      const uint32_t* __restrict__ m32s) {
    __shared__ SegJob s_jobs[LS_MAX_SLOTS];
    __shared__ uint32_t s_d[LS_MAX_SLOTS], s_near[LS_MAX_SLOTS];
    __shared__ uint32_t s_dmax; // largest d of this grid row's slots (all near) or ~0
    if (threadIdx.x == 0) s_dmax = 0;
    __syncthreads();
    if (threadIdx.x < nslots) {
        const SegJob j = jobs[threadIdx.x], j0 = jobs[0];
        s_jobs[threadIdx.x] = j;
        // slot origin Q_s = Q_0 + 6 d with 0 <= d < 2^32 (both positive)
        const bool near = !j.qneg && !j0.qneg && j.qbase >= j0.qbase && (j.qbase - j0.qbase) / 6 < (1ull << 32);
        s_near[threadIdx.x] = near;
        s_d[threadIdx.x] = near ? (uint32_t)((j.qbase - j0.qbase) / 6) : 0;
        if (threadIdx.x >= blockIdx.y * LS_GROUP && threadIdx.x < (blockIdx.y + 1) * LS_GROUP)
            atomicMax(&s_dmax, near ? s_d[threadIdx.x] : 0xFFFFFFFFu);
    }
    __syncthreads();
    const uint32_t dmax = s_dmax;
    for (uint64_t i = iL0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < iL1;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t p = primes[i];
        uint32_t m32, k00;
        if (k00s != nullptr) { // precomputed once per batch (k_large_first, k_large_m32)
            // primes above every slot offset of this row need no remainder
            // of d (d mod p = d), so their 32-bit magic is not even loaded
            m32 = p > dmax ? 0u : m32s[i - iL0];
            k00 = k00s[i - iL0];
        } else {
            const uint64_t m = m64[i];
            m32 = (uint32_t)(m >> 32); // <= floor(2^32 / p)
            k00 = first_a6(s_jobs[0], p, m);
        }
        const uint32_t c = b_shift6_cf(p);
        const uint32_t s1 = min(nslots, (blockIdx.y + 1) * LS_GROUP);
        for (uint32_t s = blockIdx.y * LS_GROUP; s < s1; ++s) {
            const SegJob& j = s_jobs[s];
            uint32_t k0;
            if (s_near[s]) {
                const uint32_t d = s_d[s];
                uint32_t r = d;
                if (d >= p) { // d mod p, quotient low by <= 2
                    r = d - __umulhi(d, m32) * p;
                    while (r >= p) r -= p;
                }
                k0 = k00 >= r ? k00 - r : k00 + (p - r);
            } else {
                k0 = first_a6(j, p, m64[i]);
            }
            const uint32_t k0b = k0 >= c ? k0 - c : k0 + (p - c);
            const uint32_t ncells = j.qg_words * 32;
            uint32_t* ga = qg + s * qg_stride_words;
            uint32_t* gb = ga + j.qg_words;
            // 32-bit steps: k < ncells < 2^32 and the step test cannot wrap
            // (p < 2^32 near the 2^64 ceiling)
            for (uint32_t k = k0; k < ncells;) {
                atomicAnd(ga + (k >> 5), ~(1u << (k & 31)));
                if (p >= ncells - k) break;
                k += p;
            }
            for (uint32_t k = k0b; k < ncells;) {
                atomicAnd(gb + (k >> 5), ~(1u << (k & 31)));
                if (p >= ncells - k) break;
                k += p;
            }
        }
    }
}

// Primes at or above the batch threshold (sparse primes: a few multiples per
// batch at most): one visit per prime and batch instead of one per grid row
// of k_large_strike.  The batch's slots are ascending and near (host-checked,
// LargeBatchTab), so every slot window is the range [d_s, d_s + nc_s) of one
// coordinate axis k (q = Q_0 + 6k) that starts at slot 0's origin.  The
// thread walks the prime's multiples k0, k0 + p, ... below the span end once
// per class array, finds the last slot with d_s <= k by a predicated scan of
// the register-resident origins, and strikes that slot and, in the halo
// overlap, the one before it (the reference's sparse-prime hit list,
// sieve.cpp:109-126, made a batch-wide walk).  No per-slot remainders, no
// per-slot loops: ~1/8 of k_large_strike's work for these primes.
__device__ __forceinline__ void lb_strike_walk(uint32_t k, uint32_t p, const LargeBatchTab& T,
                                               const uint32_t* __restrict__ s_d, const uint32_t* __restrict__ s_nc, const uint32_t* __restrict__ s_base,
                                               uint32_t* __restrict__ qg) {
    while (k < T.span) {
        uint32_t s = 0;
#pragma unroll
        for (uint32_t j = 1; j < MAX_SLOTS; ++j) s += k >= T.d[j]; // unused slots: d = ~0
        const uint32_t o = k - s_d[s];
        if (o < s_nc[s]) atomicAnd(qg + s_base[s] + (o >> 5), ~(1u << (o & 31)));
        if (s > 0) { // halo overlap with the previous slot's window
            const uint32_t o1 = k - s_d[s - 1];
            if (o1 < s_nc[s - 1]) atomicAnd(qg + s_base[s - 1] + (o1 >> 5), ~(1u << (o1 & 31)));
        }
        if (p >= T.span - k) break; // no 32-bit wrap near the 2^64 ceiling
        k += p;
    }
}

__global__ void __launch_bounds__(256) k_large_batch(const SegJob* __restrict__ jobs, LargeBatchTab T,
                                                     const uint32_t* __restrict__ primes,
                                                     const uint64_t* __restrict__ m64, uint64_t i0, uint64_t i1,
                                                     uint32_t* __restrict__ qg, uint64_t qg_stride_words) {
    // per slot: cells per class array, word offsets of arrays A and B
    __shared__ uint32_t s_d[MAX_SLOTS], s_nc[MAX_SLOTS], s_ba[MAX_SLOTS], s_bb[MAX_SLOTS];
    __shared__ SegJob s_j0;
    if (threadIdx.x < MAX_SLOTS) {
        const uint32_t s = threadIdx.x;
        s_d[s] = T.d[s];
        const uint32_t qw = s < T.n ? jobs[s].qg_words : 0;
        s_nc[s] = qw * 32;
        s_ba[s] = (uint32_t)(s * qg_stride_words);
        s_bb[s] = (uint32_t)(s * qg_stride_words) + qw;
    }
    if (threadIdx.x == 0) s_j0 = jobs[0];
    __syncthreads();
    for (uint64_t i = i0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < i1;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t p = primes[i];
        const uint32_t k0 = first_a6(s_j0, p, m64[i]);
        const uint32_t c = b_shift6_cf(p);
        const uint32_t k0b = k0 >= c ? k0 - c : k0 + (p - c);
        lb_strike_walk(k0, p, T, s_d, s_nc, s_ba, qg);
        lb_strike_walk(k0b, p, T, s_d, s_nc, s_bb, qg);
    }
}

// k_large_strike's grid rows when the batch's slots line up on one wheel axis
// (LargeBatchTab, host-checked): a row of LS_GROUP slots is one range
// [D, E) of that axis, so a prime takes ONE remainder for the row (the first
// multiple at or above D, from its batch first index k00) and walks its
// multiples through the range, striking each slot of the row whose window
// holds the cell (both, in the halo overlap).  Against the per-slot form
// this drops the per-slot remainders, folds and loop set-ups.  Rows run in
// grid order, so the REDs of one row stay in the row's L2-resident masks.
// FIRST: the launch of row 0 (D = 0), which computes each prime's batch
// first index k00 itself and stores it for the launch of the other rows (no
// separate k_large_first pass): from the previous batch's k00 when that batch
// lay dd < 2^32 wheel steps below (k00 = k00_prev - dd mod p, one 32-bit
// remainder; may alias k00s), else by the 64-bit first_a6 at slot 0's origin.  The
// prime tables stream through L2 with evict-first loads, so the row's slot
// masks stay resident for the REDs.
template <bool FIRST>
__global__ void __launch_bounds__(256) k_large_rows(LargeBatchTab T, const SegJob* __restrict__ jobs,
                                                    const uint32_t* __restrict__ primes,
                                                    const uint64_t* __restrict__ m64, uint64_t iL0, uint64_t iL1,
                                                    uint32_t* __restrict__ qg, uint64_t qg_stride_words,
                                                    uint32_t* k00s, const uint32_t* __restrict__ m32s, uint32_t row0,
                                                    const uint32_t* k00_prev, uint32_t dd) {
    static_assert(LS_GROUP == 2, "row walk written for two slots per row");
    // T.cop >= 1, s_cop bit x (x < 5005): gcd(x, 5*7*11*13) = 1.  A multiple q
    // of a large prime that 5, 7, 11 or 13 also divides is already clear in
    // the tile (the presieve), so its RED can be skipped: 42 % of the strikes
    // for two remainders per strike.  Off by default: the row walk is
    // issue-bound (72 % issue active), and the remainders cost more than the
    // REDs they save (C5 window 0.140 s off, 0.163 s at 1, 0.196 s at 2).
    __shared__ uint32_t s_cop[(5005 + 31) / 32];
    if (T.cop && threadIdx.x < (5005 + 31) / 32) {
        const uint32_t w = threadIdx.x * 32;
        // bit b of P_p set iff b mod p != 0 (b < 64); word = P_p >> (w mod p)
        constexpr uint64_t P5 = 0xEF7BDEF7BDEF7BDEull, P7 = 0x7EFDFBF7EFDFBF7Eull;
        constexpr uint64_t P11 = 0xFF7FEFFDFFBFF7FEull, P13 = 0xFFEFFF7FFBFFDFFEull;
        s_cop[threadIdx.x] = (uint32_t)(P5 >> (w % 5)) & (uint32_t)(P7 >> (w % 7)) & (uint32_t)(P11 >> (w % 11)) &
                             (uint32_t)(P13 >> (w % 13));
    }
    // s_cop2 bit x (x < 7429): gcd(x, 17*19*23) = 1 (T.cop >= 2: a further
    // 15 % of the remaining strikes for one more remainder per strike)
    __shared__ uint32_t s_cop2[(7429 + 31) / 32];
    if (T.cop >= 2 && threadIdx.x < (7429 + 31) / 32) {
        const uint32_t w = threadIdx.x * 32;
        constexpr uint64_t P17 = 0xFFF7FFFBFFFDFFFEull, P19 = 0xFDFFFFBFFFF7FFFEull, P23 = 0xFFFFBFFFFF7FFFFEull;
        s_cop2[threadIdx.x] = (uint32_t)(P17 >> (w % 17)) & (uint32_t)(P19 >> (w % 19)) &
                              (uint32_t)(P23 >> (w % 23));
    }
    __shared__ SegJob s_j0;
    if (FIRST && threadIdx.x == 0) s_j0 = jobs[0];
    __syncthreads();
    const uint32_t s0 = (row0 + blockIdx.y) * LS_GROUP;
    const bool two = s0 + 1 < T.n;
    const uint32_t D = T.d[s0];
    const uint32_t nc0 = T.qw[s0] * 32;
    const uint32_t dl = two ? T.d[s0 + 1] - D : 0;  // second slot's start within the row
    const uint32_t nc1 = two ? T.qw[s0 + 1] * 32 : 0;
    const uint32_t L = max(nc0, dl + nc1);          // row range [D, D + L)
    uint32_t* const a0 = qg + s0 * qg_stride_words; // slot s0: A, then B at + qgw
    uint32_t* const b0 = a0 + T.qw[s0];
    uint32_t* const a1 = a0 + qg_stride_words;
    uint32_t* const b1 = two ? a1 + T.qw[s0 + 1] : a1;
    for (uint64_t i = iL0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < iL1;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t p = __ldcs(primes + i);
        uint32_t k00, r = D; // r = D mod p (quotient of the 32-bit magic low by <= 2)
        if (FIRST) {
            if (k00_prev != nullptr) { // the previous batch's first index, dd wheel steps below
                const uint32_t kp = __ldcs(k00_prev + (i - iL0));
                uint32_t rd = dd;
                if (dd >= p) {
                    rd = dd - __umulhi(dd, __ldcs(m32s + (i - iL0))) * p;
                    while (rd >= p) rd -= p;
                }
                k00 = kp >= rd ? kp - rd : kp + (p - rd);
            } else {
                k00 = first_a6(s_j0, p, __ldcs(m64 + i));
            }
            __stcs(k00s + (i - iL0), k00);
        } else {
            k00 = __ldcs(k00s + (i - iL0));
            if (D >= p) {
                r = D - __umulhi(D, __ldcs(m32s + (i - iL0))) * p;
                while (r >= p) r -= p;
            }
        }
        const uint32_t oa = k00 >= r ? k00 - r : k00 + (p - r);
        const uint32_t c = b_shift6_cf(p);
        const uint32_t ob = oa >= c ? oa - c : oa + (p - c);
#pragma unroll
        for (int arr = 0; arr < 2; ++arr) {
            uint32_t* const w0 = arr ? b0 : a0;
            uint32_t* const w1 = arr ? b1 : a1;
            const uint32_t q0 = T.qm[s0][arr], q1 = T.qm[s0 + two][arr]; // slot origin (+4 for B) mod 5005
            const uint32_t r0 = T.qm2[s0][arr], r1 = T.qm2[s0 + two][arr]; // ... mod 7429
            for (uint32_t o = arr ? ob : oa; o < L;) {
                const uint32_t o1 = o - dl; // wraps above nc1 when o < dl
                bool h0 = o < nc0, h1 = o1 < nc1;
                if (T.cop) {
                    const uint32_t x = (q0 + 6 * o) % 5005u, x1 = (q1 + 6 * o1) % 5005u;
                    h0 = h0 && (s_cop[x >> 5] >> (x & 31) & 1);
                    h1 = h1 && (s_cop[x1 >> 5] >> (x1 & 31) & 1);
                    if (T.cop >= 2) {
                        const uint32_t y = (r0 + 6 * o) % 7429u, y1 = (r1 + 6 * o1) % 7429u;
                        h0 = h0 && (s_cop2[y >> 5] >> (y & 31) & 1);
                        h1 = h1 && (s_cop2[y1 >> 5] >> (y1 & 31) & 1);
                    }
                }
#ifdef GB_LS_BOUNDS // bounds probe (compute-sanitizer is unavailable on the GPU pool)
                auto inside = [&](const uint32_t* w) {
                    const uint64_t off = (uint64_t)(w - qg), s = off / qg_stride_words;
                    return s < T.n && off - s * qg_stride_words < 2ull * T.qw[s];
                };
                if (h0 && !inside(w0 + (o >> 5))) { GB_STAT(7, 1); h0 = false; }
                if (h1 && !inside(w1 + (o1 >> 5))) { GB_STAT(7, 1); h1 = false; }
#endif
                if (h0) atomicAnd(w0 + (o >> 5), ~(1u << (o & 31)));
                if (h1) atomicAnd(w1 + (o1 >> 5), ~(1u << (o1 & 31)));
                if (p >= L - o) break; // 32-bit steps cannot wrap
                o += p;
            }
        }
    }
}

// Window cells of the first strikes of {p, m, z, c'} in arrays A and B of
// the block starting at cell KB: z = k0 + p ceil(2^29 / p) (so z - KB >= 0
// for every block start), A's offset is (z - KB) mod p by the magic
// m = floor(2^32/p) (quotient low by at most one), and B's is A's + c'
// (mod p), c' = p - (4 6^-1 mod p).  Branch-free, two unsigned-min folds.
static_assert((MAX_SEG_EVENS / E6 + 1) * (uint64_t)K6 < (1ull << 29), "block starts below 2^29 cells");
__device__ __forceinline__ void block_off6(const uint4 v, uint32_t KB, uint32_t& oa, uint32_t& ob) {
    const uint32_t p = v.x;
    const uint32_t x = v.z - KB;
    const uint32_t r = x - __umulhi(x, v.y) * p;
    oa = min(r, r - p);
    const uint32_t t = oa + v.w;
    ob = min(t, t - p);
}

// ============================================================ mask fill
// Large tile primes (>= the mask threshold, default M6: at most one multiple
// per class array of a block window) are not visited block by block.  One
// CTA owns MK_CELLS consecutive cells of both class arrays of a slot's
// wheel-6 bitmask (qg) in shared memory, visits every such prime once for
// all of them (first multiple from the slot's row, then the multiples in the
// range), strikes with shared REDs and stores the words with plain coalesced
// writes: no global atomics, no hit lists.  The fused kernel ANDs the words
// of its window into the tile (sieve_block), the same words the large-prime
// strikes of k_large_strike land in (p > P_TILE_MAX, run after this).
// A block window visits a prime once per MK_CELLS / K6 = 3 blocks instead of
// once per block.
__global__ void __launch_bounds__(MK_THREADS, 1) k_mask_fill(MaskArgs A) {
    extern __shared__ __align__(16) uint32_t msm[];
    uint32_t* ma = msm;            // array A words [c0, c0 + MK_CELLS)
    uint32_t* mb = msm + MK_WORDS; // array B
    const uint32_t s = blockIdx.y;
    const uint32_t qw = A.jobs[s].qg_words;
    const uint32_t w0 = blockIdx.x * MK_WORDS;
    if (w0 >= qw) return;
    const uint32_t nw = min(MK_WORDS, qw - w0);
    const uint32_t c0 = 32 * w0, len = 32 * nw;
    for (uint32_t i = threadIdx.x; i < 2 * MK_WORDS; i += MK_THREADS) msm[i] = ~0u;
    __syncthreads();
    const uint32_t ta = (uint32_t)__cvta_generic_to_shared(ma), tb = (uint32_t)__cvta_generic_to_shared(mb);
    const uint4* rows = A.pmc + (size_t)s * A.np - A.iA0;
    auto one = [&](const uint4 v) {
        uint32_t oa, ob;
        block_off6(v, c0, oa, ob); // first multiples at or after c0, relative to it
        for (uint32_t x = oa; x < len; x += v.x)
            asm volatile("red.shared.and.b32 [%0], %1;" ::"r"(ta + ((x >> 3) & ~3u)),
                         "r"(__funnelshift_l(0xFFFFFFFEu, 0xFFFFFFFEu, x)) : "memory");
        for (uint32_t x = ob; x < len; x += v.x)
            asm volatile("red.shared.and.b32 [%0], %1;" ::"r"(tb + ((x >> 3) & ~3u)),
                         "r"(__funnelshift_l(0xFFFFFFFEu, 0xFFFFFFFEu, x)) : "memory");
    };
    // rows come from L2: MK_INFLIGHT loaded before their strikes
    uint32_t i = A.iK0 + threadIdx.x;
    for (; i + (MK_INFLIGHT - 1) * MK_THREADS < A.iK1; i += MK_INFLIGHT * MK_THREADS) {
        uint4 v[MK_INFLIGHT];
#pragma unroll
        for (int u = 0; u < MK_INFLIGHT; ++u) v[u] = __ldg(rows + i + u * MK_THREADS);
#pragma unroll
        for (int u = 0; u < MK_INFLIGHT; ++u) one(v[u]);
    }
    for (; i < A.iK1; i += MK_THREADS) one(__ldg(rows + i));
    __syncthreads();
    uint32_t* ga = A.qg + s * A.qg_stride_words + w0;
    uint32_t* gb = ga + qw;
    for (uint32_t w = threadIdx.x; w < nw; w += MK_THREADS) {
        ga[w] = ma[w];
        gb[w] = mb[w];
    }
}

// ============================================================ K2 + K3
// Wheel-6 tile: [TPAD][A: M6W words][TPAD][B: M6W words][TPAD], pads zero.
__device__ __forceinline__ uint32_t* arr_a(uint32_t* t) { return t + TPAD; }
__device__ __forceinline__ uint32_t* arr_b(uint32_t* t) { return t + 2 * TPAD + M6W; }
__device__ __forceinline__ const uint32_t* arr_a(const uint32_t* t) { return t + TPAD; }
__device__ __forceinline__ const uint32_t* arr_b(const uint32_t* t) { return t + 2 * TPAD + M6W; }

// Warp-cooperative strikes of one prime in one class array from cell o:
// lane L strikes o + L p + k 32p; 32p cells are p words, so the lane's mask
// is loop-invariant and only the word index advances.
__device__ __forceinline__ void strike_warp6(uint32_t* arr, uint32_t o, uint32_t p, uint32_t lane) {
    const uint32_t c = o + lane * p;
    if (c >= M6) return;
    const uint32_t mask = __funnelshift_l(0xFFFFFFFEu, 0xFFFFFFFEu, c);
#if GB_RED_ADDR32
    // 32-bit shared byte addresses, four REDs per trip off one pointer
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(arr);
    const uint32_t end = base + 4 * M6W;
    const uint32_t st = 4 * p; // bytes between strikes of this lane
    uint32_t a = base + 4 * (c >> 5);
    for (; a + 3 * st < end; a += 4 * st) {
        asm volatile("red.shared.and.b32 [%0], %1;" ::"r"(a), "r"(mask) : "memory");
        asm volatile("red.shared.and.b32 [%0], %1;" ::"r"(a + st), "r"(mask) : "memory");
        asm volatile("red.shared.and.b32 [%0], %1;" ::"r"(a + 2 * st), "r"(mask) : "memory");
        asm volatile("red.shared.and.b32 [%0], %1;" ::"r"(a + 3 * st), "r"(mask) : "memory");
    }
    for (; a < end; a += st) asm volatile("red.shared.and.b32 [%0], %1;" ::"r"(a), "r"(mask) : "memory");
#else
    uint32_t wi = c >> 5;
    const uint32_t p2 = 2 * p, p3 = 3 * p, p4 = 4 * p;
    for (; wi + p3 < M6W; wi += p4) {
        atomicAnd(&arr[wi], mask);
        atomicAnd(&arr[wi + p], mask);
        atomicAnd(&arr[wi + p2], mask);
        atomicAnd(&arr[wi + p3], mask);
    }
    for (; wi < M6W; wi += p) atomicAnd(&arr[wi], mask);
#endif
}

// One strike of cell c if c < M6, without a branch: single-strike primes hit a
// block with probability < 1/2, so a branch around the strike costs the warp
// its BSSY/BRA/BSYNC on every site.  A miss (c >= M6) is clamped into the
// TPAD >= 32 zero words past the array (word M6W + lane at most; distinct
// banks across the warp), where clearing a bit of a zero word is a no-op.
static_assert(TPAD >= 32, "branch-free strikes need 32 pad words past each array");
#ifndef GB_STRIKE_IMAD
#define GB_STRIKE_IMAD 1
#endif
__constant__ uint32_t c_four = 4; // not a compile-time constant: keeps (w * 4 + base) an IMAD
__constant__ uint32_t c_2p27 = 1u << 27; // likewise keeps c >> 5 an IMAD.HI (GB_STRIKE_IMAD=2)
#ifndef GB_RUN_IMAD
#define GB_RUN_IMAD 1 // run-loop strikes: word address as shift + IMAD (1e12 0.333 -> 0.328 s, 1e13 3.87 -> 3.82 s)
#endif
__device__ __forceinline__ void strike_if(uint32_t* arr, uint32_t c, uint32_t lane) {
#if GB_PRED_STRIKE == 2
    // predicated RED: a miss issues the instruction but moves no data
    (void)lane;
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(arr) + ((c >> 3) & ~3u);
    asm volatile("{\n\t.reg .pred p;\n\tsetp.lt.u32 p, %0, %1;\n\t@p red.shared.and.b32 [%2], %3;\n\t}"
                 ::"r"(c), "r"(M6), "r"(a), "r"(__funnelshift_l(0xFFFFFFFEu, 0xFFFFFFFEu, c)) : "memory");
#elif GB_PRED_STRIKE && GB_STRIKE_IMAD
    // word address as one IMAD with a constant-bank 4: the multiply runs on
    // the FMA pipe instead of a shift, mask and add on the ALU pipe (the
    // kernel's binding pipe)
    const uint32_t cc = min(c, M6 + 32 * lane);
#if GB_STRIKE_IMAD >= 2
    // cc >> 5 as the high word of cc * 2^27: IMAD.HI, also on the FMA pipe
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(arr) + __umulhi(cc, c_2p27) * c_four;
#else
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(arr) + (cc >> 5) * c_four;
#endif
    asm volatile("red.shared.and.b32 [%0], %1;" ::"r"(a), "r"(__funnelshift_l(0xFFFFFFFEu, 0xFFFFFFFEu, cc)) : "memory");
#elif GB_PRED_STRIKE
    strike(arr, min(c, M6 + 32 * lane));
#else
    if (c < M6) strike(arr, c);
#endif
}

#if GB_RUN_IMAD
// run-loop strike with the word address as shift + IMAD (FMA pipe) instead of
// shift + mask + add
__device__ __forceinline__ void strike6(uint32_t* arr, uint32_t c) {
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(arr) + (c >> 5) * c_four;
    asm volatile("red.shared.and.b32 [%0], %1;" ::"r"(a), "r"(__funnelshift_l(0xFFFFFFFEu, 0xFFFFFFFEu, c)) : "memory");
}
#elif GB_STRIKE_IMAD >= 3
// strike with the word address on the FMA pipe (IMAD.HI + IMAD)
__device__ __forceinline__ void strike6(uint32_t* arr, uint32_t c) {
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(arr) + __umulhi(c, c_2p27) * c_four;
    asm volatile("red.shared.and.b32 [%0], %1;" ::"r"(a), "r"(__funnelshift_l(0xFFFFFFFEu, 0xFFFFFFFEu, c)) : "memory");
}
#else
__device__ __forceinline__ void strike6(uint32_t* arr, uint32_t c) { strike(arr, c); }
#endif

// strikes c, c + step, ... < M6 of one class array (two per trip)
__device__ __forceinline__ void strike_run6(uint32_t* arr, uint32_t c, uint32_t step, uint32_t lane) {
    while (c + step < M6) {
        strike6(arr, c);
        strike6(arr, c + step);
        c += 2 * step;
    }
    strike_if(arr, c, lane);
}

// Thread-per-prime strikes of rows [q, qe) (stride GT), INF rows loaded
// before their strikes.  K = 0: runs of any length (strike_run6); K > 0: at
// most K strikes per array, unrolled and clamped (strike_if).
template <int GT, int K, int INF>
__device__ __forceinline__ void strike_rows(uint32_t* A6, uint32_t* B6, const uint4* q, const uint4* qe, uint32_t KB,
                                            uint32_t lane) {
    auto one = [&](const uint4 v) {
        uint32_t oa, ob;
        block_off6(v, KB, oa, ob);
        if constexpr (K == 0) {
            strike_run6(A6, oa, v.x, lane);
            strike_run6(B6, ob, v.x, lane);
        } else {
#pragma unroll
            for (int k = 0; k < K; ++k) {
                strike_if(A6, oa + k * v.x, lane);
                strike_if(B6, ob + k * v.x, lane);
            }
        }
    };
    for (; q + (INF - 1) * GT < qe; q += INF * GT) {
        uint4 v[INF];
#pragma unroll
        for (int u = 0; u < INF; ++u) v[u] = __ldg(q + u * GT);
#pragma unroll
        for (int u = 0; u < INF; ++u) one(v[u]);
    }
    for (; q < qe; q += GT) one(__ldg(q));
}

// ---- 2-CTA cluster pairing (k_verify_pair).  The CTAs of a cluster sieve
// two consecutive blocks b0 = 2j, b0 + 1 of one slot.  A prime >= M6 (>= K6)
// strikes each class array of a window at most once, and its offset in block
// b0 + 1 follows from the one in b0 with one compare: o' = o - K6 (o >= K6)
// or o + p - K6.  So each such row is visited ONCE per pair: the rows are
// interleaved between the two CTAs, and every visit strikes its own tile
// locally and the peer's tile through distributed shared memory.  mbarriers
// (arrived remotely, release/acquire at cluster scope) order the peer's
// presieve before the remote strikes, and the remote strikes before the
// peer's check reads its tile.
struct PairCtx {
    uint32_t rank;        // 0: block b0, 1: block b0 + 1
    bool own_valid;       // this CTA has a block in the pair (the last pair of an odd slot has one)
    bool peer_valid;
    uint32_t KB0;         // window start cell of b0
    uint32_t peer_tile;   // shared::cluster address of the peer's tile (same buffer)
    uint32_t peer_done;   // shared::cluster address of the peer's mb_done[buffer]
};

__device__ __forceinline__ uint32_t mapa_peer(uint32_t local_shared_addr, uint32_t peer) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_shared_addr), "r"(peer));
    return r;
}
__device__ __forceinline__ void red_and_cluster(uint32_t addr, uint32_t v) {
    asm volatile("red.shared::cluster.and.b32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// Wait for phase `parity` of a local mbarrier the peer arrives on; a
// protocol error traps after ~2^32 cycles instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait_cluster(uint32_t addr, uint32_t parity) {
    const long long t0 = clock64();
    for (;;) {
        uint32_t ok;
        asm volatile("{\n\t.reg .pred p;\n\t"
                     "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(addr), "r"(parity) : "memory");
        if (ok) return;
        if (clock64() - t0 > (1ll << 32)) __trap();
    }
}
// The whole group waits for an mbarrier phase: one warp spins, the others
// sleep at the group's named barrier (no issue slots taken from the check
// warps), then every thread acquires the completed phase (returns at once).
template <int GT>
__device__ __forceinline__ void mbar_wait_group(uint32_t addr, uint32_t parity, uint32_t tid, int bar) {
    if (tid < 32) mbar_wait_cluster(addr, parity);
    asm volatile("bar.sync %0, %1;" ::"r"(bar), "n"(GT) : "memory");
    mbar_wait_cluster(addr, parity);
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Single-strike rows [q, qe) (stride GT2 = 2 GT, this CTA's interleave) for
// both blocks of the pair: own block locally, the peer's through DSMEM.
template <int GT2, int INF>
__device__ __forceinline__ void strike_rows_pair(uint32_t* A6, uint32_t* B6, const uint4* q, const uint4* qe,
                                                 const PairCtx& P, uint32_t lane) {
    const uint32_t pa = P.peer_tile + 4 * TPAD, pb = P.peer_tile + 4 * (2 * TPAD + M6W);
    auto one = [&](const uint4 v) {
        uint32_t oa0, ob0;
        block_off6(v, P.KB0, oa0, ob0);
        const uint32_t p = v.x; // > K6
        const uint32_t oa1 = oa0 >= K6 ? oa0 - K6 : oa0 + (p - K6);
        const uint32_t ob1 = ob0 >= K6 ? ob0 - K6 : ob0 + (p - K6);
        const uint32_t oa = P.rank ? oa1 : oa0, ob = P.rank ? ob1 : ob0; // own block
        const uint32_t xa = P.rank ? oa0 : oa1, xb = P.rank ? ob0 : ob1; // peer's block
        if (P.own_valid) {
            strike_if(A6, oa, lane);
            strike_if(B6, ob, lane);
        }
#ifndef GB_PAIR_NOREMOTE // timing probe: no remote strikes (wrong results)
        if (P.peer_valid) {
            if (xa < M6) red_and_cluster(pa + ((xa >> 3) & ~3u), __funnelshift_l(0xFFFFFFFEu, 0xFFFFFFFEu, xa));
            if (xb < M6) red_and_cluster(pb + ((xb >> 3) & ~3u), __funnelshift_l(0xFFFFFFFEu, 0xFFFFFFFEu, xb));
        }
#else
        (void)xa;
        (void)xb;
#endif
    };
    for (; q + (INF - 1) * GT2 < qe; q += INF * GT2) {
        uint4 v[INF];
#pragma unroll
        for (int u = 0; u < INF; ++u) v[u] = __ldg(q + u * GT2);
#pragma unroll
        for (int u = 0; u < INF; ++u) one(v[u]);
    }
    for (; q < qe; q += GT2) one(__ldg(q));
}

// K2 strikes of one block by a group of GT threads (tid = index in the
// group): warp-cooperative below P_WARP_MAX (rows wsplit[warp][..], balanced
// by the host), one thread per prime above; primes >= M6 (index >= nW)
// strike each array at most once.  pmc: this slot's rows (index i - iA0).
template <int GT, bool PAIR = false>
__device__ __forceinline__ void strike_verify6(uint32_t* tile, const uint4* __restrict__ pmc, uint32_t nA,
                                               uint32_t nQ, uint32_t nH, uint32_t nW, uint32_t nB, uint32_t nK,
                                               uint32_t KB,
                                               uint32_t tid,
                                               const uint16_t* __restrict__ wsplit, const PairCtx* P = nullptr,
                                               uint32_t mb_ready = 0, uint32_t parity = 0, int bar = 0) {
    const uint32_t lane = tid & 31, warp = tid >> 5;
    uint32_t* A6 = arr_a(tile);
    uint32_t* B6 = arr_b(tile);
    {
        const uint32_t idx = wsplit[warp * 32 + lane];
        const uint32_t nmine = __popc(__ballot_sync(0xffffffffu, idx != 0xFFFFu)); // packed from lane 0
        uint32_t pm = 0, oam = M6, obm = M6;
        if (idx != 0xFFFFu) {
            const uint4 v = __ldg(pmc + idx);
            pm = v.x;
            block_off6(v, KB, oam, obm);
        }
        for (uint32_t k = 0; k < nmine; ++k) {
            const uint32_t oa = __shfl_sync(0xffffffffu, oam, k);
            const uint32_t ob = __shfl_sync(0xffffffffu, obm, k);
            const uint32_t p = __shfl_sync(0xffffffffu, pm, k);
            strike_warp6(A6, oa, p, lane);
            strike_warp6(B6, ob, p, lane);
        }
    }
    // thread per prime; the rows come from L2, so several are loaded before
    // their strikes to keep loads in flight per warp.  Primes >= M6/4 strike
    // an array at most 4 (>= M6/2: 2, >= M6: 1) times, unrolled branch-free.
    // rows end at nK (the first mask prime; nB when the mask fill is off)
    nQ = min(nQ, nK);
    nH = min(nH, nK);
    nW = min(nW, nK);
    nB = min(nB, nK);
    strike_rows<GT, 0, GB_RUN_INFLIGHT>(A6, B6, pmc + nA + tid, pmc + nQ, KB, lane);
    strike_rows<GT, 4, GB_RUN_INFLIGHT>(A6, B6, pmc + nQ + tid, pmc + nH, KB, lane);
    constexpr int SS_INFLIGHT = GT == 32 * WS_SW_LIGHT ? GB_SS_INFLIGHT_LIGHT : GB_SS_INFLIGHT_HEAVY;
    strike_rows<GT, 2, SS_INFLIGHT>(A6, B6, pmc + nH + tid, pmc + nW, KB, lane);
#ifndef GB_SKIP_SINGLE // timing probe: no single-strike primes (wrong results)
    if constexpr (PAIR) {
        // the peer has presieved its tile (remote strikes may start), then
        // this CTA's interleave of the rows for both blocks
        mbar_wait_group<GT>(mb_ready, parity, tid, bar);
        strike_rows_pair<2 * GT, SS_INFLIGHT>(A6, B6, pmc + nW + P->rank * GT + tid, pmc + nB, *P, lane);
    } else {
        strike_rows<GT, 1, SS_INFLIGHT>(A6, B6, pmc + nW + tid, pmc + nB, KB, lane);
    }
#else
    if constexpr (PAIR) mbar_wait_group<GT>(mb_ready, parity, tid, bar);
#endif
}

// Presieve one class array (M6W words) with the wheel-6 patterns; ph[g] =
// pattern index of the array's cell 0.  Each thread builds 4 consecutive
// words per step (one 16-B store): per group 5 loads, 4 funnel shifts.
__device__ __forceinline__ void presieve6(uint32_t* arr, const uint32_t* pat6, const uint32_t (&ph)[4], uint32_t tid,
                                          uint32_t nthr) {
    uint32_t o[4], step[4];
#pragma unroll
    for (int g = 0; g < 4; ++g) {
        o[g] = (ph[g] + 128u * tid) % pg6_p(g);
        step[g] = (128u * nthr) % pg6_p(g);
    }
    for (uint32_t wd = 4 * tid; wd < M6W; wd += 4 * nthr) {
        uint4 v = make_uint4(~0u, ~0u, ~0u, ~0u);
#pragma unroll
        for (int g = 0; g < 4; ++g) {
            const uint32_t* pg = pat6 + pg6_off(g) + (o[g] >> 5);
            const uint32_t sh = o[g];
            const uint32_t w0 = pg[0], w1 = pg[1], w2 = pg[2], w3 = pg[3], w4 = pg[4];
            v.x &= __funnelshift_r(w0, w1, sh);
            v.y &= __funnelshift_r(w1, w2, sh);
            v.z &= __funnelshift_r(w2, w3, sh);
            v.w &= __funnelshift_r(w3, w4, sh);
            const uint32_t on = o[g] + step[g];
            o[g] = min(on, on - pg6_p(g));
        }
        *reinterpret_cast<uint4*>(arr + wd) = v;
    }
}

__device__ __forceinline__ void set_cell(uint32_t* arr, uint32_t k) { atomicOr(&arr[k >> 5], 1u << (k & 31)); }
__device__ __forceinline__ void clear_cell(uint32_t* arr, uint32_t k) { atomicAnd(&arr[k >> 5], ~(1u << (k & 31))); }

// Window of a block whose origin Qs (signed) is at most sbound: q <= 1 is
// not prime, and every base prime p >= 5 inside the window (struck as a
// multiple of itself, or presieved) is restored.
__device__ __forceinline__ void fixup_low6(uint32_t* tile, int64_t Qs, const uint32_t* __restrict__ primes,
                                           uint64_t n_primes, uint64_t sbound, uint32_t tid, uint32_t nthr) {
    uint32_t* A6 = arr_a(tile);
    uint32_t* B6 = arr_b(tile);
    // cells with q <= 1 (A: Qs + 6k <= 1, B: Qs + 4 + 6k <= 1)
    if (Qs <= 1) {
        const int64_t na6 = (1 - Qs) / 6 + 1;
        const uint32_t na = na6 < (int64_t)M6 ? (uint32_t)na6 : M6;
        for (uint32_t k = tid; k < na; k += nthr) clear_cell(A6, k);
    }
    if (Qs <= -3) {
        const int64_t nb6 = (-3 - Qs) / 6 + 1;
        const uint32_t nb = nb6 < (int64_t)M6 ? (uint32_t)nb6 : M6;
        for (uint32_t k = tid; k < nb; k += nthr) clear_cell(B6, k);
    }
    // presieved primes 5..47 (their patterns clear them)
    if (tid < N_PAT_PRIMES - 1) {
        const int64_t d = (int64_t)pat_prime(tid + 1) - Qs;
        if (d >= 0 && d < 6 * (int64_t)M6) {
            if (d % 6 == 0) set_cell(A6, (uint32_t)(d / 6));
            else set_cell(B6, (uint32_t)((d - 4) / 6));
        }
    }
    // base primes in [max(Qs, 5), min(Qs + 6 M6 - 1, sbound)]
    const int64_t lo = Qs > 5 ? Qs : 5;
    const int64_t wend = Qs + 6 * (int64_t)M6 - 1;
    const int64_t hi = wend < (int64_t)sbound ? wend : (int64_t)sbound;
    if (lo > hi) return;
    uint64_t a = 0, b = n_primes; // first index with primes[i] >= lo
    while (a < b) {
        const uint64_t m = (a + b) >> 1;
        if ((int64_t)primes[m] < lo) a = m + 1; else b = m;
    }
    for (uint64_t i = a + tid; i < n_primes; i += nthr) {
        const int64_t p = primes[i];
        if (p > hi) break;
        const int64_t d = p - Qs;
        if (d % 6 == 0) set_cell(A6, (uint32_t)(d / 6));
        else set_cell(B6, (uint32_t)((d - 4) / 6));
    }
}

// 64 cells [x - 64, x) of a class array as a u64 (bit 63 <-> cell x - 1);
// x may be as low as 64 - 32 TPAD (the leading pad reads as zeros).
__device__ __forceinline__ uint64_t window6(const uint32_t* arr, int32_t x) {
    const int32_t lo = x - 64;
    const int32_t wi = lo >> 5;
    const uint32_t sh = (uint32_t)lo & 31;
    const uint32_t w0 = arr[wi], w1 = arr[wi + 1], w2 = arr[wi + 2];
    return ((uint64_t)__funnelshift_r(w1, w2, sh) << 32) | __funnelshift_r(w0, w1, sh);
}
__device__ __forceinline__ bool cell6(const uint32_t* arr, int32_t k) { return (arr[k >> 5] >> (k & 31)) & 1; }

// Per-thread K3 accumulators of one block (sums wrap mod 2^64).
struct K3Acc {
    uint64_t sp = 0;          // sum p
    uint64_t spi = 0;         // sum p * il (il = even index within the block)
    uint32_t mp = 0;          // max p over per-even (deep / generic) evens
    uint32_t mi = 0xFFFFFFFFu; // its smallest il
    __device__ __forceinline__ void observe(uint32_t p, uint32_t il) {
        if (p > mp || (p == mp && il < mi)) {
            mp = p;
            mi = il;
        }
    }
    __device__ __forceinline__ void add(uint32_t p, uint32_t il) {
        sp += p;
        spi += (uint64_t)p * il;
        observe(p, il);
    }
};

// Candidates p <= PBS are scanned bit-sliced (gb_bitslice.cuh bs6_scan_r*),
// 32 class-r evens per lane; the few evens left ("deep") continue per even
// over 64-wide windows of g = p div 6, from the first window with an
// unscanned candidate.
constexpr uint32_t PBS = BS6_PMAX;
// first deep window per class: the first window with an unscanned candidate
constexpr uint32_t DEEP_J0_R0 = ((BS6_PMAX_R0 + 1) / 6) / 64;
constexpr uint32_t DEEP_J0_R24 = ((BS6_PMAX_R24 + 1) / 6) / 64;
__device__ __forceinline__ uint32_t deep_j0(uint32_t r) { return r == 0 ? DEEP_J0_R0 : DEEP_J0_R24; }
constexpr int NPL = BS6_PLANES;          // z planes
#ifndef GB_QCAP
#define GB_QCAP 128 // 512 before the 1.5 x 2^18 tile (equal speed at 256 / 128)
#endif
constexpr uint32_t QCAP = GB_QCAP;       // per-warp deep-even queue (classes 2, 4 run ~2x the mean deep rate)

// Straggler entry for an even with no candidate inside the in-tile halo.
__device__ __forceinline__ void push_straggler(const VerifyArgs& A, const SegJob& J, uint32_t s, uint32_t iseg,
                                               uint32_t jlim_small, uint32_t extra_flags) {
    const uint64_t n = J.a + 2ull * iseg;
    const uint64_t jq = (n - 6) >> 1;
    const uint64_t jmax = jq < jlim_small ? jq : jlim_small;
    const uint32_t flags = ((uint64_t)JH <= jmax ? F_NEED_P1 : F_P1_FAIL) | extra_flags;
    const unsigned idx = atomicAdd(A.list_count, 1u);
    if (idx < A.list_cap) A.list[idx] = StragEntry{s, iseg, (uint32_t)JH, flags};
    GB_STAT(4, 1);
}

// Per-class constants of a block: class ci holds the evens il = ci + 3t;
// their n = r (mod 6), and candidate g reads cell t + G - g.
struct Class6 {
    uint32_t r, G;
};
__device__ __forceinline__ Class6 class6(const SegJob& J, uint32_t ci) {
    return Class6{(uint32_t)((J.a + 2 * ci) % 6), (J.delta + 2 * ci) / 6};
}
// the three classes of a block, looked up without local memory: r and G of
// class ci follow from a mod 6 and delta (two registers, not six)
struct Classes6 {
    uint32_t a6, delta;
    __device__ __forceinline__ explicit Classes6(const SegJob& J) : a6((uint32_t)(J.a % 6)), delta(J.delta) {}
    __device__ __forceinline__ Class6 operator[](uint32_t ci) const {
        uint32_t r = a6 + 2 * ci;
        r = r >= 6 ? r - 6 : r;
        return Class6{r, (delta + 2 * ci) / 6};
    }
};

// Window j (g in [64j, 64j + 64)) of a class-r even t: smallest p with a hit
// under the masks (0 = none).  r = 2: A, p = 6g + 1; r = 4: B, p = 6g - 1;
// r = 0: A with p = 6g + 5 and B with p = 6g + 1.  lim1 / lim5 narrow the
// masks (generic path).  The first read is selected, not branched, so a warp
// whose entries mix classes does not walk every class's path.
__device__ __forceinline__ uint32_t window_hit6(const uint32_t* tile, const uint64_t* masks6, uint32_t r, uint32_t G,
                                               uint32_t t, uint32_t j, uint64_t lim1, uint64_t lim5m, uint64_t lim5p) {
    const int32_t x = (int32_t)(t + G) - 64 * (int32_t)j + 1;
    const uint32_t cls = r == 2 ? 0u : r == 4 ? 1u : 2u; // masks6 row: 6g+1, 6g-1, 6g+5
    const uint64_t lim = r == 2 ? lim1 : r == 4 ? lim5m : lim5p;
    const int32_t off = r == 2 ? 1 : r == 4 ? -1 : 5;
    const uint64_t m = window6(r == 4 ? arr_b(tile) : arr_a(tile), x) & masks6[cls * NWIN6 + j] & lim;
    uint32_t p = m ? (uint32_t)(6 * (int32_t)(64 * j + __clzll(m)) + off) : 0xFFFFFFFFu;
    if (r == 0) {
        const uint64_t mb = window6(arr_b(tile), x) & masks6[j] & lim1;
        if (mb) p = min(p, 6 * (64 * j + __clzll(mb)) + 1);
    }
    return p == 0xFFFFFFFFu ? 0 : p;
}

// Deep even of a fast block in place (queue overflow): windows j0 .. NWIN6-1.
template <bool PMIN>
__device__ __forceinline__ void deep_even6(const uint32_t* tile, const uint64_t* masks6, uint32_t t, const Class6 C,
                                           uint32_t ci, uint32_t i0, uint32_t s, const SegJob& J,
                                           const VerifyArgs& A, uint32_t jlim_small, K3Acc& acc) {
    GB_STAT(1, 1);
    uint32_t p = 0;
    for (uint32_t j = deep_j0(C.r); j < (uint32_t)NWIN6 && !p; ++j)
        p = window_hit6(tile, masks6, C.r, C.G, t, j, ~0ull, ~0ull, ~0ull);
    const uint32_t il = ci + 3 * t;
    if (p) acc.add(p, il);
    else push_straggler(A, J, s, i0 + il, jlim_small, 0);
    if constexpr (PMIN) A.pmin_out[i0 + il] = p;
}

// One round over the warp's deep-even queue: the top n entries
// (t | ci << DQ_CI | j << DQ_J) each test ONE window j; misses are pushed back
// with j + 1, so no lane idles while another walks many windows.
template <bool PMIN>
__device__ __forceinline__ uint32_t deep_round6(const uint32_t* tile, const uint64_t* masks6, uint32_t* q, uint32_t qn,
                                                uint32_t n, uint32_t lane, uint32_t i0, uint32_t s, const SegJob& J,
                                                const Classes6& CL, const VerifyArgs& A, uint32_t jlim_small,
                                                K3Acc& acc) {
    qn -= n;
    const bool act = lane < n;
    const uint32_t e = act ? q[qn + lane] : 0u;
    __syncwarp();
    if (lane == 0) GB_STAT(3, 1);
    bool again = false;
    if (act) {
        const uint32_t t = e & ((1u << DQ_CI) - 1), ci = (e >> DQ_CI) & 3u, j = e >> DQ_J;
        const Class6 C = CL[ci];
        const uint32_t p = window_hit6(tile, masks6, C.r, C.G, t, j, ~0ull, ~0ull, ~0ull);
        const uint32_t il = ci + 3 * t;
        if (p) {
            acc.add(p, il);
            if constexpr (PMIN) A.pmin_out[i0 + il] = p;
        } else if (j + 1 < (uint32_t)NWIN6) {
            again = true;
        } else {
            push_straggler(A, J, s, i0 + il, jlim_small, 0);
            if constexpr (PMIN) A.pmin_out[i0 + il] = 0;
        }
    }
    const uint32_t bal = __ballot_sync(0xffffffffu, again);
    if (again) q[qn + __popc(bal & ((1u << lane) - 1))] = e + (1u << DQ_J);
    __syncwarp();
    return qn + __popc(bal);
}

#ifndef GB_DQ_WORDS
#define GB_DQ_WORDS 1 // deep queue of word entries (0: one entry per even)
#endif
// Word-entry deep queue (GB_DQ_WORDS): one two-word entry per lane-word with
// deep evens, {U = its unresolved evens, (t0 + 32) | ci << DQ_CI | j << DQ_J}
// with t0 = the word's first class index.  Appending takes one ballot per
// word step instead of a prefix over count thresholds and a per-even store
// loop.  A round takes n entries; each tests ONE window j of its lowest
// unresolved even.  A hit (or a straggler after the last window) clears that
// even and restarts j at the class's first deep window for the next one;
// a miss moves to window j + 1.  Entries with evens left go back.
static_assert(QCAP >= 128, "word entries: < 32 queued + 32 appended <= QCAP / 2");
template <bool PMIN>
__device__ __forceinline__ uint32_t deep_round6w(const uint32_t* tile, const uint64_t* masks6, uint32_t* q,
                                                 uint32_t qn, uint32_t n, uint32_t lane, uint32_t i0, uint32_t s,
                                                 const SegJob& J, const Classes6& CL, const VerifyArgs& A,
                                                 uint32_t jlim_small, K3Acc& acc) {
    qn -= n;
    const bool act = lane < n;
    uint32_t U = act ? q[2 * (qn + lane)] : 0u;
    uint32_t e = act ? q[2 * (qn + lane) + 1] : 0u;
    __syncwarp();
    if (lane == 0) GB_STAT(3, 1);
    if (act) {
        const uint32_t bit = __ffs(U) - 1;
        const uint32_t t = (e & ((1u << DQ_CI) - 1)) - 32 + bit, ci = (e >> DQ_CI) & 3u;
        uint32_t j = e >> DQ_J;
        const Class6 C = CL[ci];
        const uint32_t p = window_hit6(tile, masks6, C.r, C.G, t, j, ~0ull, ~0ull, ~0ull);
        const uint32_t il = ci + 3 * t;
        if (p) {
            acc.add(p, il);
            if constexpr (PMIN) A.pmin_out[i0 + il] = p;
            U &= U - 1;
            j = deep_j0(C.r);
        } else if (j + 1 < (uint32_t)NWIN6) {
            ++j;
        } else {
            push_straggler(A, J, s, i0 + il, jlim_small, 0);
            if constexpr (PMIN) A.pmin_out[i0 + il] = 0;
            U &= U - 1;
            j = deep_j0(C.r);
        }
        e = (e & ((1u << DQ_J) - 1)) | (j << DQ_J);
    }
    const bool again = U != 0;
    const uint32_t bal = __ballot_sync(0xffffffffu, again);
    if (again) {
        const uint32_t k = qn + __popc(bal & ((1u << lane) - 1));
        q[2 * k] = U;
        q[2 * k + 1] = e;
    }
    __syncwarp();
    return qn + __popc(bal);
}

// bits m of window j with g = 64j + m <= gl (bit 63 - m)
__device__ __forceinline__ uint64_t glim_mask(int64_t gl, uint32_t j) {
    const int64_t mm = gl - 64 * (int64_t)j;
    if (mm < 0) return 0;
    if (mm >= 63) return ~0ull;
    return ~0ull << (63 - mm);
}

// Generic per-even check (windows near the start of the number line, small
// p_small, injected even): candidates p <= min(p_small, n - 3, PH6) in
// ascending order, then the straggler list.
template <bool PMIN>
__device__ __forceinline__ void generic_even6(const uint32_t* tile, const uint64_t* masks6, uint32_t il,
                                              uint32_t i0, uint32_t s, const SegJob& J, const VerifyArgs& A,
                                              uint32_t jlim_small, K3Acc& acc) {
    const uint32_t iseg = i0 + il;
    const uint64_t n = J.a + 2ull * iseg;
    uint32_t p = 0;
    if (n == 4) {
        p = 2;
    } else {
        const uint32_t ci = il % 3, t = il / 3;
        const Class6 C = class6(J, ci);
        uint64_t pmax = n - 3;
        if (pmax > A.p_small) pmax = A.p_small;
        if (pmax > PH6) pmax = PH6;
        if (pmax >= 3) {
            if (n == 6) p = 3; // q = 3 has no cell
            else if (C.r == 2 && cell6(arr_b(tile), (int32_t)(t + C.G) - 1)) p = 3;
            else if (C.r == 4 && cell6(arr_a(tile), (int32_t)(t + C.G))) p = 3;
        }
        if (!p && pmax >= 5) {
            const int64_t g1 = ((int64_t)pmax - 1) / 6, g5m = ((int64_t)pmax + 1) / 6, g5p = ((int64_t)pmax - 5) / 6;
            for (uint32_t j = 0; j < (uint32_t)NWIN6 && !p; ++j) {
                if (64 * (int64_t)j > g5m) break;
                p = window_hit6(tile, masks6, C.r, C.G, t, j, glim_mask(g1, j), glim_mask(g5m, j),
                                pmax >= 5 ? glim_mask(g5p, j) : 0);
            }
        }
        if (!p) push_straggler(A, J, s, iseg, jlim_small, n == A.inject ? F_INJECT : 0u);
    }
    if (p) {
        acc.add(p, il);
        if (n == A.inject) {
            const unsigned idx = atomicAdd(A.list_count, 1u);
            if (idx < A.list_cap) A.list[idx] = StragEntry{s, iseg, 0u, F_INJECT | F_OBSERVED};
        }
    }
    if constexpr (PMIN) A.pmin_out[iseg] = p;
}

// sum of the bit indices set in x
__device__ __forceinline__ uint32_t idx_sum(uint32_t x) {
    return __popc(x & 0xAAAAAAAAu) + 2 * __popc(x & 0xCCCCCCCCu) + 4 * __popc(x & 0xF0F0F0F0u) +
           8 * __popc(x & 0xFF00FF00u) + 16 * __popc(x & 0xFFFF0000u);
}

// Deferred sum p * (bit index) of VFLUSH words: V = bit-sliced per-position
// sums of z (VPL planes), FC = per-position found counts (FPL planes);
// p = 3 + 2z, so the sum is 2 sum_b 2^b idx(V_b) + 3 sum_k 2^k idx(FC_k).
// Resets V and FC.
// words per vertical-counter reduction: longer batches amortise the flush
// but widen the counters (registers); the check group's size decides
#ifndef GB_VFLUSH_LIGHT
#define GB_VFLUSH_LIGHT 24 // 16 check warps: 24 steps per class with the 1.5 x 2^18 tile, one flush
#endif
#ifndef GB_VFLUSH_HEAVY
#define GB_VFLUSH_HEAVY 22 // 12 check warps: 22 steps per class, one flush
#endif
__host__ __device__ constexpr int ilog2c(uint32_t x) { return x <= 1 ? 0 : 1 + ilog2c((x + 1) / 2); } // ceil(log2 x)
__host__ __device__ constexpr int vpl_of(uint32_t vf) { return NPL + ilog2c(vf); } // vf (2^NPL - 1) < 2^vpl
#if BS6_CODE
// class code c: p = 3c + kf F + ke Z0 (gen_bitslice.py class_code), and
// kf F + ke Z0 = sg (g0 + 2 g1) with g0 = F & ~Z0, g1 = Z0 (class 0) or 0,
// sg = -1 for class 4, else +1.  FC counts g0 + 2 g1 per position.
__host__ __device__ constexpr int fpl_of(uint32_t vf) { return ilog2c(2 * vf + 1); } // 2 vf < 2^fpl
template <int VPL, int FPL>
__device__ __forceinline__ uint32_t vsum_by_index(uint32_t (&V)[VPL], uint32_t (&FC)[FPL], uint32_t sg) {
    uint32_t qv = 0, qf = 0;
#pragma unroll
    for (int b = 0; b < VPL; ++b) {
        qv += (1u << b) * idx_sum(V[b]);
        V[b] = 0;
    }
#pragma unroll
    for (int k = 0; k < FPL; ++k) {
        qf += (1u << k) * idx_sum(FC[k]);
        FC[k] = 0;
    }
    return 3 * qv + sg * qf; // mod 2^32: the sum itself is < 2^32
}
#else
__host__ __device__ constexpr int fpl_of(uint32_t vf) { return ilog2c(vf + 1); } // vf < 2^fpl
template <int VPL, int FPL>
__device__ __forceinline__ uint32_t vsum_by_index(uint32_t (&V)[VPL], uint32_t (&FC)[FPL], uint32_t) {
    uint32_t q = 0;
#pragma unroll
    for (int b = 0; b < VPL; ++b) {
        q += (2u << b) * idx_sum(V[b]);
        V[b] = 0;
    }
#pragma unroll
    for (int k = 0; k < FPL; ++k) {
        q += (3u << k) * idx_sum(FC[k]);
        FC[k] = 0;
    }
    return q;
}
#endif

// p of plane code c in class r
__device__ __forceinline__ uint32_t code_p(uint32_t r, uint32_t c) {
#if BS6_CODE
    const uint32_t o = c & 1;
    return r == 0 ? 3 * c + 1 + o : r == 2 ? 3 * c + 1 - o : 3 * c - 1 + o;
#else
    return 3 + 2 * c;
#endif
}

// Per-class constants of the word sums (code mode): p = 3c + kf F + ke Z0.
struct ClassSums {
    uint32_t kz0;  // weight of popc(Z0) beyond 3: 3 + ke
    uint32_t kf;   // weight of popc(F) (two's complement)
    uint32_t g1m;  // g1 = Z0 & g1m
    uint32_t sg;   // sign of the FC counter (two's complement)
};
__device__ __forceinline__ ClassSums class_sums(uint32_t r) {
    ClassSums S;
    S.kz0 = r == 2 ? 2u : 4u;
    S.kf = r == 4 ? 0xFFFFFFFFu : 1u;
    S.g1m = r == 0 ? ~0u : 0u;
    S.sg = r == 4 ? 0xFFFFFFFFu : 1u;
    return S;
}

// The tile words a scan reads, WB - BS6_WORDS + 1 .. WB of each array (4 up
// to candidate ~ 6 * 95, 3 for the lower bounds of 7-plane builds).
#if BS6_NWORDS == 4
#define BS6_LOAD_WORDS(a, b)                                                  \
    const uint32_t a0 = a[-3], a1 = a[-2], a2 = a[-1], a3 = a[0];             \
    const uint32_t b0 = b[-3], b1 = b[-2], b2 = b[-1], b3 = b[0]
#define BS6_ARGS a0, a1, a2, a3, b0, b1, b2, b3
#elif BS6_NWORDS == 3
#define BS6_LOAD_WORDS(a, b)                                                  \
    const uint32_t a0 = a[-2], a1 = a[-1], a2 = a[0];                         \
    const uint32_t b0 = b[-2], b1 = b[-1], b2 = b[0]
#define BS6_ARGS a0, a1, a2, b0, b1, b2
#else
#error "scan words per array: 3 or 4"
#endif

// Bit-sliced scan of word w of class r: U in = valid evens of the word,
// U out = those with no candidate p <= PBS; Z = planes of the found z.
__device__ __forceinline__ void scan_word6(const uint32_t* tile, uint32_t r, uint32_t WB, uint32_t& U,
                                           uint32_t (&Z)[NPL]) {
    const uint32_t* a = arr_a(tile) + WB;
    const uint32_t* b = arr_b(tile) + WB;
    BS6_LOAD_WORDS(a, b);
    if (r == 0) bs6_scan_r0(BS6_ARGS, U, Z);
    else if (r == 2) bs6_scan_r2(BS6_ARGS, U, Z);
    else bs6_scan_r4(BS6_ARGS, U, Z);
}

// Sums of one scanned word: sum p (weighted by the word's even index), and
// its z planes / found bits into the vertical counters.
template <bool PMIN, int VPL, int FPL>
__device__ __forceinline__ void word_sums(const VerifyArgs& A, uint32_t w, uint32_t valid, uint32_t U,
                                          const uint32_t (&Z)[NPL], uint32_t ci, uint32_t delta, uint32_t i0,
                                          uint32_t (&V)[VPL], uint32_t (&FC)[FPL], uint32_t& sp32, K3Acc& acc,
                                          const ClassSums& CS, uint32_t r) {
    const uint32_t F = valid & ~U;
#if BS6_CODE
    // p = 3c + kf F + ke Z0: sum p of the word; il = ci + 3 (32w - delta + i)
    uint32_t P = CS.kf * __popc(F) + CS.kz0 * __popc(Z[0]);
#pragma unroll
    for (int bp = 1; bp < NPL; ++bp) P += (3u << bp) * __popc(Z[bp]);
#else
    // p = 3 + 2z: sum p of the word; il = ci + 3 (32w - delta + i)
    uint32_t P = 3 * __popc(F);
#pragma unroll
    for (int bp = 0; bp < NPL; ++bp) P += (2u << bp) * __popc(Z[bp]);
#endif
    sp32 += P;
    acc.spi += (uint64_t)P * (uint64_t)((int64_t)ci + 96 * (int64_t)w - 3 * (int64_t)delta);
    // V += Z, FC += F (ripple-carry, bit-sliced)
    uint32_t cy = V[0] & Z[0];
    V[0] ^= Z[0];
#pragma unroll
    for (int bp = 1; bp < NPL; ++bp) {
        const uint32_t v = V[bp], z = Z[bp];
        V[bp] = v ^ z ^ cy;
        cy = (v & z) | (cy & (v ^ z));
    }
#pragma unroll
    for (int bp = NPL; bp < VPL; ++bp) {
        const uint32_t v = V[bp];
        V[bp] = v ^ cy;
        cy = v & cy;
    }
#if BS6_CODE
    {
        // FC += g0 + 2 g1 (g1 only in class 0)
        const uint32_t g0 = F & ~Z[0], g1 = Z[0] & CS.g1m;
        const uint32_t f0 = FC[0];
        FC[0] = f0 ^ g0;
        const uint32_t c0 = f0 & g0;
        const uint32_t f1 = FC[1];
        FC[1] = f1 ^ g1 ^ c0;
        cy = (f1 & g1) | (c0 & (f1 ^ g1));
#pragma unroll
        for (int kk = 2; kk < FPL; ++kk) {
            const uint32_t f = FC[kk];
            FC[kk] = f ^ cy;
            cy = f & cy;
        }
    }
#else
    cy = F;
#pragma unroll
    for (int kk = 0; kk < FPL; ++kk) {
        const uint32_t f = FC[kk];
        FC[kk] = f ^ cy;
        cy = f & cy;
    }
#endif
    if constexpr (PMIN) {
        for (uint32_t i = 0; i < 32; ++i) {
            if (!((F >> i) & 1)) continue;
            uint32_t z = 0;
#pragma unroll
            for (int bp = 0; bp < NPL; ++bp) z |= ((Z[bp] >> i) & 1) << bp;
            A.pmin_out[i0 + ci + 3 * (32 * w - delta + i)] = code_p(r, z);
        }
    }
}

// Scan + sums of one word of class R (compile-time class: the per-class sum
// constants become immediates).  Returns U (the deep evens).
template <bool PMIN, uint32_t R, int VPL, int FPL>
__device__ __forceinline__ uint32_t scan_sums(const VerifyArgs& A, const uint32_t* tile, uint32_t WB, uint32_t w,
                                              uint32_t valid, uint32_t ci, uint32_t delta, uint32_t i0,
                                              uint32_t (&V)[VPL], uint32_t (&FC)[FPL], uint32_t& sp32, K3Acc& acc) {
    const uint32_t* a = arr_a(tile) + WB;
    const uint32_t* b = arr_b(tile) + WB;
    BS6_LOAD_WORDS(a, b);
    uint32_t U = valid, Z[NPL];
    if constexpr (R == 0) bs6_scan_r0(BS6_ARGS, U, Z);
    else if constexpr (R == 2) bs6_scan_r2(BS6_ARGS, U, Z);
    else bs6_scan_r4(BS6_ARGS, U, Z);
    ClassSums CS;
    CS.kz0 = R == 2 ? 2u : 4u;
    CS.kf = R == 4 ? 0xFFFFFFFFu : 1u;
    CS.g1m = R == 0 ? ~0u : 0u;
    CS.sg = R == 4 ? 0xFFFFFFFFu : 1u;
    word_sums<PMIN, VPL, FPL>(A, w, valid, U, Z, ci, delta, i0, V, FC, sp32, acc, CS, R);
    return U;
}

// Deep evens of one word (U): appended to the warp's round queue, positions
// from a ballot per count threshold (counts are 0..2 almost always); full
// rounds run as soon as 32 entries wait.  Warp-uniform call.
template <bool PMIN>
__device__ __forceinline__ uint32_t word_deep(const uint32_t* tile, const uint64_t* masks6, uint32_t* q, uint32_t qn,
                                              uint32_t U, uint32_t w, uint32_t ci, uint32_t delta, const Class6 C,
                                              uint32_t lane, uint32_t i0, uint32_t s, const SegJob& J,
                                              const Classes6& CL, const VerifyArgs& A, uint32_t jlim_small,
                                              K3Acc& acc) {
#if GB_DQ_WORDS
    const uint32_t m = __ballot_sync(0xffffffffu, U != 0);
    if (m == 0) return qn;
#ifdef GB_STATS
    const uint32_t tot = __reduce_add_sync(0xffffffffu, __popc(U));
    if (lane == 0) GB_STAT(2, tot);
#endif
    const uint32_t ne = __popc(m);
    if (qn + ne <= QCAP / 2) {
        if (U) {
            const uint32_t k = qn + __popc(m & ((1u << lane) - 1));
            q[2 * k] = U;
            q[2 * k + 1] = (32 * w - delta + 32) | (ci << DQ_CI) | (deep_j0(C.r) << DQ_J);
        }
        qn += ne;
        __syncwarp();
        while (qn >= 32) qn = deep_round6w<PMIN>(tile, masks6, q, qn, 32, lane, i0, s, J, CL, A, jlim_small, acc);
    } else {
        while (U) { // queue full (cannot happen with QCAP >= 128): in place
            const uint32_t bit = __ffs(U) - 1;
            U &= U - 1;
            deep_even6<PMIN>(tile, masks6, 32 * w - delta + bit, C, ci, i0, s, J, A, jlim_small, acc);
        }
        __syncwarp();
    }
    return qn;
#endif
    const uint32_t cnt = __popc(U);
    const uint32_t cmax = __reduce_max_sync(0xffffffffu, cnt);
    if (cmax == 0) return qn;
    const uint32_t total = __reduce_add_sync(0xffffffffu, cnt);
    const uint32_t lt = (1u << lane) - 1;
    uint32_t pre = 0;
    for (uint32_t th = 1; th <= cmax; ++th) pre += __popc(__ballot_sync(0xffffffffu, cnt >= th) & lt);
    if (lane == 0) GB_STAT(2, total);
    if (qn + total <= QCAP) {
        uint32_t pos = qn + pre;
        const uint32_t t0 = 32 * w - delta; // wraps for w = 0; t0 + bit >= 0 for valid bits
        const uint32_t hi = (ci << DQ_CI) | (deep_j0(C.r) << DQ_J);
        while (U) {
            const uint32_t bit = __ffs(U) - 1;
            U &= U - 1;
            q[pos++] = (t0 + bit) | hi;
        }
        qn += total;
        __syncwarp();
        while (qn >= 32) qn = deep_round6<PMIN>(tile, masks6, q, qn, 32, lane, i0, s, J, CL, A, jlim_small, acc);
    } else {
        while (U) { // queue full: this lane's deep evens in place
            const uint32_t bit = __ffs(U) - 1;
            U &= U - 1;
            deep_even6<PMIN>(tile, masks6, 32 * w - delta + bit, C, ci, i0, s, J, A, jlim_small, acc);
        }
        __syncwarp();
    }
    return qn;
}

// Valid bits of word w of a class with T evens and alignment delta.
__device__ __forceinline__ uint32_t word_mask6(uint32_t w, uint32_t T, uint32_t delta) {
    uint32_t m = ~0u;
    if (w == 0) m <<= delta;
    const int64_t hi = (int64_t)T + delta - 32 * (int64_t)w; // bits < hi valid
    if (hi < 32) m &= hi <= 0 ? 0u : (1u << hi) - 1;
    return m;
}

// Barrier of one group of GT threads.
template <int GT>
__device__ __forceinline__ void gbar(int id) { asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(GT) : "memory"); }
__device__ __forceinline__ void nb_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void nb_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// Where flat block fb of a batch lies: slot, block of the slot, window.
struct BlockInfo {
    SegJob J;
    uint32_t s, b;  // slot, block index within the slot
    uint32_t KB;    // window start cell relative to the slot's origin (b K6)
    bool low;       // window origin <= sbound: fix-up needed
    int64_t Qs;     // window origin (valid when low)
};

__device__ __forceinline__ BlockInfo block_info(const VerifyArgs& A, const SegJob* jobs, uint32_t fb) {
    BlockInfo I;
    uint32_t s = 0; // few slots: linear scan
    while (s + 1 < A.nslots && jobs[s + 1].block_prefix <= fb) ++s;
    I.s = s;
    I.J = jobs[s];
    I.b = fb - I.J.block_prefix;
    I.KB = I.b * K6;
    const uint64_t off = 6ull * I.KB;
    if (I.J.qneg) {
        I.Qs = (int64_t)off - (int64_t)I.J.qbase;
        I.low = I.Qs <= (int64_t)A.sbound;
    } else {
        I.low = I.J.qbase <= A.sbound && off <= A.sbound - I.J.qbase;
        I.Qs = I.low ? (int64_t)(I.J.qbase + off) : 0;
    }
    return I;
}

// K2: sieve block I into tile by one group (tid = index in the group).  On
// return this thread's strikes and fix-ups are issued; the caller's barrier
// publishes them.
template <int GT, bool PAIR = false>
__device__ __forceinline__ void sieve_block(const VerifyArgs& A, uint32_t* tile, const uint32_t* pat6,
                                            const BlockInfo& I, uint32_t tid, int bar, const PairCtx* P = nullptr,
                                            uint32_t mb_ready = 0, uint32_t mb_done = 0, uint32_t peer_ready = 0,
                                            uint32_t parity = 0) {
    if constexpr (PAIR) {
        if (!P->own_valid) {
            // no block of our own in this pair (the last pair of a slot with
            // an odd block count): our share of the peer's single-strike
            // rows and the handshakes only
            mbar_arrive_remote(peer_ready);
            mbar_wait_group<GT>(mb_ready, parity, tid, bar);
            const uint32_t nB = min(A.iB1, A.iK0) - A.iA0, nW = min(A.iW1 - A.iA0, nB);
            const uint4* pmc = A.pmc + (size_t)I.s * A.np;
            constexpr int SS_INFLIGHT = GT == 32 * WS_SW_LIGHT ? GB_SS_INFLIGHT_LIGHT : GB_SS_INFLIGHT_HEAVY;
            strike_rows_pair<2 * GT, SS_INFLIGHT>(arr_a(tile), arr_b(tile), pmc + nW + P->rank * GT + tid, pmc + nB,
                                                  *P, tid & 31);
            mbar_arrive_remote(P->peer_done);
            mbar_wait_group<GT>(mb_done, parity, tid, bar);
            return;
        }
    }
    uint32_t pha[4], phb[4];
#pragma unroll
    for (int g = 0; g < 4; ++g) {
        const uint32_t P = pg6_p(g), iv = inv6_mod(P);
        const uint32_t qm = (uint32_t)((I.J.qmod[g] + 6ull * (I.KB % P)) % P); // Q_b mod P
        pha[g] = (uint32_t)((uint64_t)((qm + P - 1) % P) * iv % P);            // (Q_b - 1)/6
        phb[g] = (uint32_t)((uint64_t)((qm + 3) % P) * iv % P);                // (Q_b + 3)/6
    }
    presieve6(arr_a(tile), pat6, pha, tid, GT);
    presieve6(arr_b(tile), pat6, phb, tid, GT);
    gbar<GT>(bar);
    if constexpr (PAIR) mbar_arrive_remote(peer_ready); // our presieve is visible: the peer may strike into us
    if (A.qg != nullptr && I.J.qg_words) {
        // large-prime mask words of this window (k_mask_fill, k_large_strike),
        // ANDed as REDs so they need no barrier against the strikes below
        const uint32_t* ga = A.qg + I.s * A.qg_stride_words + I.KB / 32;
        const uint32_t* gb = ga + I.J.qg_words;
        const uint32_t lim = min(M6W, I.J.qg_words - I.KB / 32);
        const uint32_t sa = (uint32_t)__cvta_generic_to_shared(arr_a(tile));
        const uint32_t sb = (uint32_t)__cvta_generic_to_shared(arr_b(tile));
        constexpr int U = 4;
        uint32_t wd = tid;
        for (; wd + (U - 1) * GT < lim; wd += U * GT) {
            uint32_t va[U], vb[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                va[u] = __ldcs(ga + wd + u * GT);
                vb[u] = __ldcs(gb + wd + u * GT);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                asm volatile("red.shared.and.b32 [%0], %1;" ::"r"(sa + 4 * (wd + u * GT)), "r"(va[u]) : "memory");
                asm volatile("red.shared.and.b32 [%0], %1;" ::"r"(sb + 4 * (wd + u * GT)), "r"(vb[u]) : "memory");
            }
        }
        for (; wd < lim; wd += GT) {
            asm volatile("red.shared.and.b32 [%0], %1;" ::"r"(sa + 4 * wd), "r"(__ldcs(ga + wd)) : "memory");
            asm volatile("red.shared.and.b32 [%0], %1;" ::"r"(sb + 4 * wd), "r"(__ldcs(gb + wd)) : "memory");
        }
    }
#ifndef GB_SKIP_STRIKES // timing probe: the check group on presieved-only tiles
    strike_verify6<GT, PAIR>(tile, A.pmc + (size_t)I.s * A.np, A.iA1 - A.iA0, A.iQ1 - A.iA0, A.iH1 - A.iA0,
                             A.iW1 - A.iA0, A.iB1 - A.iA0, A.iK0 - A.iA0, I.KB, tid,
                             A.wsplit, P, mb_ready, parity, bar);
#else
    if constexpr (PAIR) mbar_wait_group<GT>(mb_ready, parity, tid, bar);
#endif
    if constexpr (PAIR) {
        // our remote strikes into the peer are issued (release), and the
        // peer's into us are complete before the fix-up and the check
        mbar_arrive_remote(P->peer_done);
        mbar_wait_group<GT>(mb_done, parity, tid, bar);
    }
    if (I.low) {
        gbar<GT>(bar);
        fixup_low6(tile, I.Qs, A.primes, A.n_primes, A.sbound, tid, GT);
    }
}

// K3: minimal p of every even of block I over the sieved tile, by one group;
// the block's sums / max key go to the slot accumulators.
template <bool PMIN, int GT>
__device__ __forceinline__ void check_block(const VerifyArgs& A, const uint32_t* tile, const uint64_t* masks6,
                                            const BlockInfo& I, uint32_t tid, uint32_t (*s_q)[QCAP]) {
    const uint32_t lane = tid & 31, warp = tid >> 5;
    const uint32_t jlim_small = A.p_small >= 3 ? (uint32_t)min((A.p_small - 3) / 2, (uint64_t)0xFFFFFFFFu) : 0;
    const uint32_t s = I.s;
    const SegJob& J = I.J;
    const uint32_t i0 = I.b * E6;
    const uint32_t ne = min(E6, J.evens - i0);
    const uint64_t n_first = J.a + 2ull * i0, n_last = n_first + 2ull * (ne - 1);
    const bool inject_here = (A.inject & 1) == 0 && A.inject >= n_first && A.inject <= n_last;
    // fast blocks: every even has all candidates p <= PH6 valid (n >= PH6 + 3,
    // p_small >= PH6), no n = 4, no injected even
    const bool fast = n_first >= PH6 + 3 && jlim_small >= (uint32_t)JH - 1 && !inject_here;
    K3Acc acc;
    if (fast && tid == 0) GB_STAT(5, 1);
    if (fast) {
        uint32_t* q = s_q[warp];
        uint32_t qn = 0;   // warp-uniform queue length (< 32 between batches)
        uint32_t sp32 = 0; // sum p of the bit-sliced evens (< 2^32 per lane)
        // sum p * (bit index) is deferred: z planes and found bits of VFLUSH
        // words are summed per bit position as bit-sliced counters V (z) and
        // FC (found), then reduced by bit index once
        constexpr uint32_t VFLUSH = GT >= 512 ? GB_VFLUSH_LIGHT : GB_VFLUSH_HEAVY;
        constexpr int VPL = vpl_of(VFLUSH), FPL = fpl_of(VFLUSH);
        uint32_t V[VPL], FC[FPL];
#pragma unroll
        for (int k = 0; k < VPL; ++k) V[k] = 0;
#pragma unroll
        for (int k = 0; k < FPL; ++k) FC[k] = 0;
        const Classes6 CL(J);
        uint32_t nbatch = 0; // batches in the vertical counters
        for (uint32_t ci = 0; ci < 3; ++ci) {
            const Class6 C = CL[ci];
            const ClassSums CS = class_sums(C.r);
            const uint32_t T = ne > ci ? (ne - ci + 2) / 3 : 0;
            const uint32_t delta = C.G & 31;
            const uint32_t nw = (T + delta + 31) >> 5;
            // one word (32 class-ci evens) per lane per step; the scan is not
            // unrolled (code size: the three class scans must stay in the
            // instruction cache)
            for (uint32_t wb = warp * 32; wb < nw; wb += GT) {
                const uint32_t w = wb + lane;
                uint32_t U = 0;
                if (w < nw) {
                    const uint32_t valid = (w == 0 || w + 1 == nw) ? word_mask6(w, T, delta) : ~0u;
                    U = valid;
#if GB_CLASS_TEMPLATE
                    // scan + sums with the class constants as immediates
                    if (C.r == 0) U = scan_sums<PMIN, 0, VPL, FPL>(A, tile, w + (C.G >> 5), w, valid, ci, delta, i0, V, FC, sp32, acc);
                    else if (C.r == 2) U = scan_sums<PMIN, 2, VPL, FPL>(A, tile, w + (C.G >> 5), w, valid, ci, delta, i0, V, FC, sp32, acc);
                    else U = scan_sums<PMIN, 4, VPL, FPL>(A, tile, w + (C.G >> 5), w, valid, ci, delta, i0, V, FC, sp32, acc);
#else
                    uint32_t Z[NPL];
                    scan_word6(tile, C.r, w + (C.G >> 5), U, Z);
                    word_sums<PMIN, VPL, FPL>(A, w, valid, U, Z, ci, delta, i0, V, FC, sp32, acc, CS, C.r);
#endif
                }
                if (++nbatch == VFLUSH) { // counters hold VFLUSH words
                    acc.spi += 3ull * vsum_by_index(V, FC, CS.sg);
                    nbatch = 0;
                }
                qn = word_deep<PMIN>(tile, masks6, q, qn, U, w, ci, delta, C, lane, i0, s, J, CL, A, jlim_small, acc);
            }
#if BS6_CODE
            // the counters' weights are per class: flush at the class end
            if (nbatch) {
                acc.spi += 3ull * vsum_by_index(V, FC, CS.sg);
                nbatch = 0;
            }
#endif
        }
#if GB_DQ_WORDS
        while (qn) qn = deep_round6w<PMIN>(tile, masks6, q, qn, min(qn, 32u), lane, i0, s, J, CL, A, jlim_small, acc);
#else
        while (qn) qn = deep_round6<PMIN>(tile, masks6, q, qn, min(qn, 32u), lane, i0, s, J, CL, A, jlim_small, acc);
#endif
        if (nbatch) acc.spi += 3ull * vsum_by_index(V, FC, 1u);
        acc.sp += sp32;
    } else {
        if (tid == 0) GB_STAT(6, 1);
        if (tid == 0) GB_STAT(0, ne);
#ifndef GB_NO_GENERIC
        for (uint32_t il = tid; il < ne; il += GT) generic_even6<PMIN>(tile, masks6, il, i0, s, J, A, jlim_small, acc);
#endif
    }
    // ---- per-warp reduction -> slot accumulators; key = p << 32 | ~iseg.
    // No block barrier: sums are added per warp, and the max is taken per
    // warp (global atomicMax), so a warp never waits for the others.
    uint64_t key = acc.mp ? (((uint64_t)acc.mp << 32) | (0xFFFFFFFFu - (i0 + acc.mi))) : 0;
    uint64_t sp64 = acc.sp, spi = acc.spi + (uint64_t)i0 * acc.sp;
    for (int o = 16; o; o >>= 1) {
        sp64 += __shfl_xor_sync(0xffffffffu, sp64, o);
        spi += __shfl_xor_sync(0xffffffffu, spi, o);
        const uint64_t ok = __shfl_xor_sync(0xffffffffu, key, o);
        key = ok > key ? ok : key;
    }
    if (fast && key < ((uint64_t)(PBS + 2) << 32)) {
        // no deep even of this warp beat the bit-sliced range: its max may be
        // a bit-sliced even -- rescan its own words (w = tid mod GT, as in the
        // fast loop) for the max code (smallest il on ties)
        uint32_t bz = 0, bi = 0xFFFFFFFFu;
        for (uint32_t ci = 0; ci < 3; ++ci) {
            const Class6 C = class6(J, ci);
            const uint32_t T = ne > ci ? (ne - ci + 2) / 3 : 0;
            const uint32_t delta = C.G & 31;
            const uint32_t nw = (T + delta + 31) >> 5;
            for (uint32_t w = tid; w < nw; w += GT) {
                const uint32_t valid = word_mask6(w, T, delta);
                uint32_t U = valid, Z[NPL];
                scan_word6(tile, C.r, w + (C.G >> 5), U, Z);
                uint32_t cand = valid & ~U;
                if (!cand) continue;
                uint32_t mz = 0;
#pragma unroll
                for (int bp = NPL - 1; bp >= 0; --bp) {
                    const uint32_t tt = cand & Z[bp];
                    if (tt) {
                        cand = tt;
                        mz |= 1u << bp;
                    }
                }
                const uint32_t il = ci + 3 * (32 * w - delta + __ffs(cand) - 1);
                const uint32_t mp = code_p(C.r, mz); // codes are monotone in p within a class
                if (bi == 0xFFFFFFFFu || mp > bz || (mp == bz && il < bi)) {
                    bz = mp;
                    bi = il;
                }
            }
        }
        uint64_t kf = bi != 0xFFFFFFFFu ? (((uint64_t)bz << 32) | (0xFFFFFFFFu - (i0 + bi))) : 0;
        for (int o = 16; o; o >>= 1) {
            const uint64_t ok = __shfl_xor_sync(0xffffffffu, kf, o);
            kf = ok > kf ? ok : kf;
        }
        key = kf > key ? kf : key;
    }
    if (lane == 0) {
        atomicAdd(&A.acc[s].sum, (unsigned long long)sp64);
        atomicAdd(&A.acc[s].hash, (unsigned long long)((J.a >> 1) * sp64 + spi));
        if (key) atomicMax(&A.acc[s].key, (unsigned long long)key);
    }
}

// L2 prefetch (TMA bulk prefetch, nothing to wait for) of the large-prime
// mask words block fb's sieve will AND in: 2 x M6W words per array.  One thread.
__device__ __forceinline__ void prefetch_mask(const VerifyArgs& A, const SegJob* jobs, uint32_t fb) {
    if (fb >= A.total_blocks) return;
    uint32_t s = 0;
    while (s + 1 < A.nslots && jobs[s + 1].block_prefix <= fb) ++s;
    const SegJob& J = jobs[s];
    const uint32_t w0 = (fb - J.block_prefix) * (K6 / 32);
    if (w0 >= J.qg_words) return;
    const uint32_t bytes = 4 * min(M6W, J.qg_words - w0);
    const uint32_t* ga = A.qg + s * A.qg_stride_words + w0;
#pragma unroll
    for (int arr = 0; arr < 2; ++arr) {
        // 16-B aligned sub-range of the words (never past them: the
        // allocation's end is never crossed)
        const uint64_t a0 = reinterpret_cast<uint64_t>(ga + arr * J.qg_words);
        const uint64_t p0 = a0 & ~15ull, p1 = (a0 + bytes) & ~15ull;
        if (p1 > p0)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p0), "r"((uint32_t)(p1 - p0)) : "memory");
    }
}

// Warp-specialised fused kernel: one 896-thread CTA per SM, two wheel-6
// tile buffers.  The first 32 SW threads (the sieve group) sieve block k
// into buffer k & 1 while the other threads (the check group) check
// block k - 1 in the other buffer.  Named barriers hand buffers over:
// FULL[b] (sieve arrives, check waits) and EMPTY[b] (check arrives, sieve
// waits), so the atomic-heavy sieve and the ALU-heavy check overlap instead
// of alternating at CTA barriers.
constexpr int BAR_S = 1, BAR_FULL = 3, BAR_EMPTY = 5; // FULL/EMPTY + buffer (the check group has no internal barrier)

template <bool PMIN, int SW>
__global__ void __launch_bounds__(WS_THREADS, 1) k_verify_ws(VerifyArgs A) {
    constexpr int ST = 32 * SW, CT = WS_THREADS - ST; // sieve / check threads
    extern __shared__ __align__(16) uint32_t smem[];
    uint32_t* tiles = smem;                                 // 2 x TILE6_WORDS
    uint32_t* pat6 = smem + WS_PAT_OFF;                     // PAT6_WORDS
    uint64_t* masks6 = (uint64_t*)(smem + WS_MASK_OFF);     // 3 x NWIN6
    __shared__ uint32_t s_fb[2];
    __shared__ uint32_t s_q[CT / 32][QCAP];

    for (uint32_t i = threadIdx.x; i < PAT6_WORDS; i += blockDim.x) pat6[i] = A.gpat6[i];
    for (uint32_t i = threadIdx.x; i < 3u * NWIN6; i += blockDim.x) masks6[i] = A.masks6[i];
    // the batch's jobs (block lookup at every block start reads them)
    __shared__ SegJob s_jobs[MAX_SLOTS];
    static_assert(sizeof(SegJob) % 4 == 0, "word copy");
    for (uint32_t i = threadIdx.x; i < A.nslots * (uint32_t)(sizeof(SegJob) / 4); i += blockDim.x)
        reinterpret_cast<uint32_t*>(s_jobs)[i] = reinterpret_cast<const uint32_t*>(A.jobs)[i];
    for (uint32_t i = threadIdx.x; i < 2 * TILE6_WORDS; i += blockDim.x) tiles[i] = 0; // pads stay zero
    __syncthreads();
    const int NB = WS_THREADS; // participants of FULL / EMPTY
    if (threadIdx.x < ST) {
        // ---- sieve group.  Claims run two blocks ahead, so the mask words
        // of the block after the current one are prefetched into L2 a whole
        // block before the sieve ANDs them in.
        const uint32_t tid = threadIdx.x;
        uint32_t fb_next = 0, fb_next2 = 0;
        if (tid == 0) {
            fb_next = atomicAdd(A.block_counter, 1u);
            fb_next2 = atomicAdd(A.block_counter, 1u);
            if (A.qg != nullptr) {
                prefetch_mask(A, s_jobs, fb_next);
                prefetch_mask(A, s_jobs, fb_next2);
            }
        }
        for (uint32_t k = 0;; ++k) {
            const uint32_t bs = k & 1;
            uint32_t* tile = tiles + bs * TILE6_WORDS;
            if (k >= 2) nb_sync(BAR_EMPTY + bs, NB); // check group done with block k - 2
            if (tid == 0) s_fb[bs] = fb_next;
            gbar<ST>(BAR_S);
            const uint32_t fb = s_fb[bs];
            if (fb >= A.total_blocks) {
                if (k >= 1) nb_sync(BAR_EMPTY + (bs ^ 1), NB); // absorb the last EMPTY
                nb_arrive(BAR_FULL + bs, NB);                  // check group sees the end
                return;
            }
            if (tid == 0) {
                fb_next = fb_next2;
                fb_next2 = atomicAdd(A.block_counter, 1u);
                if (A.qg != nullptr && k > 0) prefetch_mask(A, s_jobs, fb_next);
            }
            const BlockInfo I = block_info(A, s_jobs, fb);
            sieve_block<ST>(A, tile, pat6, I, tid, BAR_S);
            if (A.tile_out != nullptr && fb == A.tile_fb) { // parity hook (gb_debug_tile)
                gbar<ST>(BAR_S);
                for (uint32_t w = tid; w < M6W; w += ST) {
                    A.tile_out[w] = arr_a(tile)[w];
                    A.tile_out[M6W + w] = arr_b(tile)[w];
                }
            }
            nb_arrive(BAR_FULL + bs, NB);
        }
    } else {
        // ---- check group
        const uint32_t tid = threadIdx.x - ST;
        for (uint32_t k = 0;; ++k) {
            const uint32_t bs = k & 1;
            nb_sync(BAR_FULL + bs, NB);
            const uint32_t fb = s_fb[bs];
            if (fb >= A.total_blocks) return;
            const BlockInfo I = block_info(A, s_jobs, fb);
#ifndef GB_SKIP_CHECK // timing probe: sieve group alone
            check_block<PMIN, CT>(A, tiles + bs * TILE6_WORDS, masks6, I, tid, s_q);
#endif
            nb_arrive(BAR_EMPTY + bs, NB);
        }
    }
}

// Paired variant of k_verify_ws: 2-CTA clusters, one block pair (b0, b0+1)
// of a slot per cluster step, claimed by rank 0 and handed to rank 1 through
// its shared memory.  Each CTA keeps the two-buffer sieve/check pipeline of
// k_verify_ws; only the single-strike rows are shared (strike_rows_pair).
// Flat block markers in s_fb: a block index, BLK_NONE (no block of ours in
// this pair: the check group skips it) or BLK_END.
constexpr uint32_t BLK_NONE = 0xFFFFFFFEu, BLK_END = 0xFFFFFFFFu;

template <bool PMIN, int SW>
__global__ void __launch_bounds__(WS_THREADS, 1) k_verify_pair(VerifyArgs A) {
    constexpr int ST = 32 * SW, CT = WS_THREADS - ST;
    extern __shared__ __align__(16) uint32_t smem[];
    uint32_t* tiles = smem;
    uint32_t* pat6 = smem + WS_PAT_OFF;
    uint64_t* masks6 = (uint64_t*)(smem + WS_MASK_OFF);
    __shared__ uint32_t s_fb[2];
    __shared__ uint32_t s_pair[2];                   // claims from rank 0
    __shared__ __align__(8) uint64_t mb_ready[2], mb_done[2], mb_claim[2];
    __shared__ uint32_t s_q[CT / 32][QCAP];
    __shared__ SegJob s_jobs[MAX_SLOTS];
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const uint32_t peer = rank ^ 1u;

    for (uint32_t i = threadIdx.x; i < PAT6_WORDS; i += blockDim.x) pat6[i] = A.gpat6[i];
    for (uint32_t i = threadIdx.x; i < 3u * NWIN6; i += blockDim.x) masks6[i] = A.masks6[i];
    for (uint32_t i = threadIdx.x; i < A.nslots * (uint32_t)(sizeof(SegJob) / 4); i += blockDim.x)
        reinterpret_cast<uint32_t*>(s_jobs)[i] = reinterpret_cast<const uint32_t*>(A.jobs)[i];
    for (uint32_t i = threadIdx.x; i < 2 * TILE6_WORDS; i += blockDim.x) tiles[i] = 0;
    if (threadIdx.x == 0) {
        for (int b = 0; b < 2; ++b) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&mb_ready[b])), "r"(ST));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&mb_done[b])), "r"(ST));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&mb_claim[b])), "r"(1));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    cluster_sync_all(); // both CTAs' barriers initialised before any remote arrive
    const int NB = WS_THREADS;
    if (threadIdx.x < ST) {
        // ---- sieve group
        const uint32_t tid = threadIdx.x;
        for (uint32_t k = 0;; ++k) {
            const uint32_t bs = k & 1, parity = (k >> 1) & 1;
            uint32_t* tile = tiles + bs * TILE6_WORDS;
            if (k >= 2) nb_sync(BAR_EMPTY + bs, NB);
            // claim pair k (rank 0) and hand it to rank 1
            if (tid == 0) {
                if (rank == 0) {
                    const uint32_t pr = atomicAdd(A.pair_counter, 1u);
                    s_pair[bs] = pr;
                    const uint32_t rp = mapa_peer((uint32_t)__cvta_generic_to_shared(&s_pair[bs]), peer);
                    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(rp), "r"(pr) : "memory");
                    mbar_arrive_remote(mapa_peer((uint32_t)__cvta_generic_to_shared(&mb_claim[bs]), peer));
                } else {
                    mbar_wait_cluster((uint32_t)__cvta_generic_to_shared(&mb_claim[bs]), parity);
                }
                // pair -> own flat block
                const uint32_t pr = s_pair[bs];
                uint32_t fb = BLK_END;
                if (pr < A.total_pairs) {
                    uint32_t s = 0;
                    while (s + 1 < A.nslots && s_jobs[s + 1].pair_prefix <= pr) ++s;
                    const uint32_t b = 2 * (pr - s_jobs[s].pair_prefix) + rank;
                    fb = b < s_jobs[s].nblocks ? s_jobs[s].block_prefix + b : BLK_NONE;
                }
                s_fb[bs] = fb;
            }
            gbar<ST>(BAR_S);
            const uint32_t fb = s_fb[bs];
            if (fb == BLK_END) {
                if (k >= 1) nb_sync(BAR_EMPTY + (bs ^ 1), NB); // absorb the last EMPTY
                nb_arrive(BAR_FULL + bs, NB);                  // check group sees the end
                break;
            }
            // the pair's first block and whether each side has one
            const uint32_t pr = s_pair[bs];
            uint32_t s = 0;
            while (s + 1 < A.nslots && s_jobs[s + 1].pair_prefix <= pr) ++s;
            const uint32_t b0 = 2 * (pr - s_jobs[s].pair_prefix);
            PairCtx P;
            P.rank = rank;
            P.own_valid = b0 + rank < s_jobs[s].nblocks;
            P.peer_valid = b0 + peer < s_jobs[s].nblocks;
            P.KB0 = b0 * K6;
            P.peer_tile = mapa_peer((uint32_t)__cvta_generic_to_shared(tile), peer);
            P.peer_done = mapa_peer((uint32_t)__cvta_generic_to_shared(&mb_done[bs]), peer);
            const uint32_t peer_ready = mapa_peer((uint32_t)__cvta_generic_to_shared(&mb_ready[bs]), peer);
            const BlockInfo I = block_info(A, s_jobs, s_jobs[s].block_prefix + b0 + (P.own_valid ? rank : 0));
            sieve_block<ST, true>(A, tile, pat6, I, tid, BAR_S, &P, (uint32_t)__cvta_generic_to_shared(&mb_ready[bs]),
                                  (uint32_t)__cvta_generic_to_shared(&mb_done[bs]), peer_ready, parity);
            if (A.tile_out != nullptr && fb == A.tile_fb) {
                gbar<ST>(BAR_S);
                for (uint32_t w = tid; w < M6W; w += ST) {
                    A.tile_out[w] = arr_a(tile)[w];
                    A.tile_out[M6W + w] = arr_b(tile)[w];
                }
            }
            nb_arrive(BAR_FULL + bs, NB);
        }
    } else {
        // ---- check group
        const uint32_t tid = threadIdx.x - ST;
        for (uint32_t k = 0;; ++k) {
            const uint32_t bs = k & 1;
            nb_sync(BAR_FULL + bs, NB);
            const uint32_t fb = s_fb[bs];
            if (fb == BLK_END) break;
            if (fb != BLK_NONE) {
                const BlockInfo I = block_info(A, s_jobs, fb);
#ifndef GB_SKIP_CHECK
                check_block<PMIN, CT>(A, tiles + bs * TILE6_WORDS, masks6, I, tid, s_q);
#endif
            }
            nb_arrive(BAR_EMPTY + bs, NB);
        }
    }
    cluster_sync_all(); // no CTA leaves while its peer may still address its shared memory
}

// ============================================================ K4
// One CTA per straggler entry: ascending candidate scan in rounds of
// blockDim.x odd p; the smallest hit of the first round with a hit wins.
__device__ uint64_t scan_min_prime(uint64_t n, uint64_t p_first, uint64_t p_last) {
    // smallest odd prime p in [p_first, p_last] with n - p prime; 0 if none
    __shared__ unsigned long long s_best;
    if ((p_first & 1) == 0) ++p_first;
    for (uint64_t r0 = p_first; r0 <= p_last; r0 += 2ull * blockDim.x) {
        if (threadIdx.x == 0) s_best = ~0ull;
        __syncthreads();
        uint64_t p = r0 + 2ull * threadIdx.x;
        if (p <= p_last && p >= r0 && is_prime_u64_dev(p) && is_prime_u64_dev(n - p))
            atomicMin(&s_best, (unsigned long long)p);
        __syncthreads();
        uint64_t best = s_best;
        __syncthreads();
        if (best != ~0ull) return best;
        if (r0 > ~0ull - 2ull * blockDim.x) break; // no wrap
    }
    return 0;
}

__global__ void k_stragglers(const SegJob* __restrict__ jobs, const StragEntry* __restrict__ list,
                             const unsigned int* __restrict__ list_count, uint32_t list_cap,
                             uint64_t p_small, StragResult* __restrict__ res,
                             uint64_t* pmin_out) {
    uint32_t cnt = min(*list_count, list_cap);
    for (uint32_t e = blockIdx.x; e < cnt; e += gridDim.x) {
        StragEntry en = list[e];
        const SegJob& J = jobs[en.slot];
        uint64_t n = J.a + 2ull * en.i_seg;
        uint64_t p1 = 0, p2 = 0;
        bool p1_failed = (en.flags & F_P1_FAIL) != 0;
        if (en.flags & F_NEED_P1) {
            // Phase 1 continuation: odd primes p in [3 + 2*j_next, min(p_small, n-3)]
            uint64_t pf = 3 + 2ull * en.j_next;
            uint64_t pl = min(p_small, n - 3);
            if (pf <= pl) p1 = scan_min_prime(n, pf, pl);
            p1_failed = p1 == 0;
        }
        if (p1_failed && !(en.flags & F_INJECT)) {
            // Phase 2: every prime <= min(p_small, n-3) failed (and p = 2 only
            // works for n = 4), so continue with primes > p_small, p <= n/2
            uint64_t pf = p_small + 1;
            uint64_t pl = n / 2;
            if (pf <= pl) p2 = scan_min_prime(n, pf, pl);
        }
        if (threadIdx.x == 0) {
            res[e] = StragResult{p1, p2};
            if (pmin_out && p1) pmin_out[en.i_seg] = p1;
        }
    }
}

// Standalone phase2_resolve (verifier.cpp:129-165) for one n.
__global__ void k_phase2_one(uint64_t n, uint64_t* out) {
    uint64_t half = n / 2;
    __shared__ uint64_t s_p;
    if (threadIdx.x == 0) s_p = (2 <= half && is_prime_u64_dev(n - 2)) ? 2 : 0;
    __syncthreads();
    uint64_t r = s_p;
    if (r == 0 && half >= 3) r = scan_min_prime(n, 3, half);
    if (threadIdx.x == 0) *out = r;
}

__global__ void k_is_prime_batch(const uint64_t* __restrict__ v, uint8_t* __restrict__ out, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = is_prime_u64_dev(v[i]) ? 1 : 0;
}

// ============================================================ finalize
// One thread: merge tile accumulators and straggler results into records.
__device__ void observe(DevRecord& r, uint64_t p, uint64_t n) {
    r.pmin_sum += p;
    r.pmin_hash += p * (n >> 1);
    if (p > r.max_p || (p == r.max_p && r.max_p != 0 && n < r.max_n)) {
        r.max_p = p;
        r.max_n = n;
    }
}

__device__ void add_ce(DevRecord& r, uint64_t n) {
    // keep the smallest GB_REC_MAX_CE ascending
    uint64_t k = r.n_ce < GB_REC_MAX_CE ? r.n_ce : GB_REC_MAX_CE;
    while (k > 0 && r.ce[k - 1] > n) {
        if (k < GB_REC_MAX_CE) r.ce[k] = r.ce[k - 1];
        --k;
    }
    if (k < GB_REC_MAX_CE) r.ce[k] = n;
    r.n_ce++;
}

__global__ void k_finalize(const SegJob* __restrict__ jobs, uint32_t nslots, const SlotAcc* __restrict__ acc,
                           const StragEntry* __restrict__ list, const unsigned int* __restrict__ list_count,
                           uint32_t list_cap, const StragResult* __restrict__ res, DevRecord* __restrict__ out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    uint32_t cnt = *list_count;
    for (uint32_t s = 0; s < nslots; ++s) {
        DevRecord r{};
        const SegJob& J = jobs[s];
        r.a = J.a;
        r.b = J.b;
        r.evens = J.evens;
        r.pmin_sum = acc[s].sum;
        r.pmin_hash = acc[s].hash;
        if (acc[s].key) {
            uint64_t k = acc[s].key;
            r.max_p = k >> 32;
            r.max_n = J.a + 2ull * (0xFFFFFFFFu - (uint32_t)(k & 0xFFFFFFFFu));
        }
        r.overflow = cnt > list_cap;
        out[s] = r;
    }
    uint32_t m = min(cnt, list_cap);
    for (uint32_t e = 0; e < m; ++e) {
        StragEntry en = list[e];
        DevRecord& r = out[en.slot];
        uint64_t n = jobs[en.slot].a + 2ull * en.i_seg;
        if (en.flags & F_OBSERVED) { // injected, Phase 1 certified in-tile
            r.unverified++;
            add_ce(r, n);
            continue;
        }
        uint64_t p1 = res[e].p1, p2 = res[e].p2;
        if (p1) observe(r, p1, n);
        if (en.flags & F_INJECT) {
            r.unverified++;
            add_ce(r, n);
            continue;
        }
        if (p1) continue;
        r.unverified++;
        if (p2) {
            r.phase2++;
            observe(r, p2, n);
        } else {
            add_ce(r, n);
        }
    }
}

// m64[i] = floor(2^64 / p_i) (p odd > 1, so = floor((2^64 - 1) / p_i))
__global__ void k_prime_magic64(const uint32_t* __restrict__ primes, uint64_t n, uint64_t* __restrict__ m64) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        m64[i] = ~0ull / primes[i];
}

// ============================================================ smem peak
// Conflict-free 128-bit shared-memory loads from every resident warp: the
// measured roofline denominator of the fused kernel (128 B/clk/SM nominal).
__global__ void __launch_bounds__(SMEM_PEAK_THREADS, 2) k_smem_peak(uint32_t iters, uint32_t* sink) {
    extern __shared__ __align__(16) uint4 sbuf[]; // 64 KiB
    constexpr uint32_t N = 4096;
    for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) sbuf[i] = make_uint4(i, i * 3, i * 5, i * 7);
    __syncthreads();
    uint32_t x = 0, y = 0, z = 0, w = 0;
    const uint32_t idx = threadIdx.x;
    for (uint32_t it = 0; it < iters; ++it) {
#pragma unroll 8
        for (uint32_t u = 0; u < 8; ++u) {
            // warp-uniform offset, consecutive lanes: conflict-free
            const uint4 v = sbuf[(idx + (it * 8 + u) * 32) & (N - 1)];
            x ^= v.x;
            y += v.y;
            z ^= v.z;
            w += v.w;
        }
    }
    if ((x ^ y ^ z ^ w) == 0x9e3779b9u) sink[blockIdx.x] = x; // keep the loads
}

// ============================================================ launchers
int debug_stats(unsigned long long* out, int reset) {
#ifdef GB_STATS
    if (cudaMemcpyFromSymbol(out, g_stats, sizeof(g_stats)) != cudaSuccess) return 1;
    if (reset) {
        unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        cudaMemcpyToSymbol(g_stats, z, sizeof(z));
    }
    return 0;
#else
    for (int i = 0; i < 8; ++i) out[i] = 0;
    (void)reset;
    return 2;
#endif
}

cudaError_t launch_smem_peak(uint32_t iters, uint32_t* sink, int grid, cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_smem_peak, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
        attr = true;
    }
    k_smem_peak<<<grid, SMEM_PEAK_THREADS, 65536, st>>>(iters, sink);
    return cudaGetLastError();
}
cudaError_t launch_init_tables(uint32_t* pat, uint32_t* pat6, uint64_t* masks6, uint64_t p_small, cudaStream_t st) {
    k_init_tables<<<64, 256, 0, st>>>(pat, pat6, masks6, p_small);
    return cudaGetLastError();
}
cudaError_t launch_seed_primes(uint32_t lim, uint32_t* out, uint32_t* count, cudaStream_t st) {
    k_seed_primes<<<1, 1024, 0, st>>>(lim, out, count);
    return cudaGetLastError();
}
cudaError_t launch_sieve_interval(uint64_t lo, uint64_t n_cells, const uint32_t* primes, uint32_t iA0,
                                  uint32_t iA1, uint32_t iB1, const uint32_t* pat, uint32_t* out,
                                  int grid, cudaStream_t st) {
    k_sieve_interval<<<grid, THREADS, SIEVE_SMEM, st>>>(lo, n_cells, primes, iA0, iA1, iB1, pat, out);
    return cudaGetLastError();
}
cudaError_t launch_count_words(const uint32_t* bits, uint64_t n_words, uint32_t chunk, uint32_t* counts,
                               uint64_t n_chunks, cudaStream_t st) {
    k_count_words<<<(unsigned)n_chunks, 256, 0, st>>>(bits, n_words, chunk, counts);
    return cudaGetLastError();
}
cudaError_t launch_scan(const uint32_t* counts, uint64_t n, uint64_t* offsets, uint64_t* total,
                        cudaStream_t st) {
    k_scan<<<1, 1024, 0, st>>>(counts, n, offsets, total);
    return cudaGetLastError();
}
cudaError_t launch_compact(const uint32_t* bits, uint64_t n_words, uint32_t chunk, const uint64_t* offsets,
                           uint64_t lo, uint32_t* primes, uint64_t n_chunks, cudaStream_t st) {
    k_compact<<<(unsigned)n_chunks, 256, 0, st>>>(bits, n_words, chunk, offsets, lo, primes);
    return cudaGetLastError();
}
cudaError_t launch_prime_magic64(const uint32_t* primes, uint64_t n, uint64_t* m64, cudaStream_t st) {
    if (!n) return cudaSuccess;
    unsigned grid = (unsigned)std::min<uint64_t>((n + 255) / 256, 148ull * 16);
    k_prime_magic64<<<grid, 256, 0, st>>>(primes, n, m64);
    return cudaGetLastError();
}
cudaError_t launch_segment_offsets(const SegJob* jobs, uint32_t nslots, const uint32_t* primes,
                                   const uint64_t* m64, uint32_t iA0, uint32_t np, uint4* pmc, cudaStream_t st) {
    if (!np || !nslots) return cudaSuccess;
    const unsigned gx = (unsigned)std::min<uint64_t>((np + 255) / 256, 148ull * 4);
    k_segment_offsets<<<dim3(gx, nslots), 256, 0, st>>>(jobs, nslots, primes, m64, iA0, np, pmc);
    return cudaGetLastError();
}
cudaError_t launch_large_strike(const SegJob* jobs, uint32_t nslots, const uint32_t* primes, const uint64_t* m64,
                                uint64_t iL0, uint64_t iL1, uint32_t* qg, uint64_t qg_stride_words, uint32_t* k00,
                                const uint32_t* m32, const LargeBatchTab* T, const uint32_t* k00_prev, uint32_t dd,
                                int* nlaunch, cudaStream_t st) {
    *nlaunch = 0;
    const uint64_t np = iL1 - iL0;
    if (!np || !nslots) return cudaSuccess;
    if (nslots > LS_MAX_SLOTS) return cudaErrorInvalidValue;
    const unsigned gx = (unsigned)std::min<uint64_t>((np + 255) / 256, 148ull * 16);
    if (T != nullptr && k00 != nullptr && m32 != nullptr) { // slots on one axis: the row walk
        const unsigned rows = (nslots + LS_GROUP - 1) / LS_GROUP;
        k_large_rows<true><<<dim3(gx, 1), 256, 0, st>>>(*T, jobs, primes, m64, iL0, iL1, qg, qg_stride_words, k00, m32, 0,
                                                        k00_prev, dd);
        *nlaunch = 1;
        if (rows > 1) {
            k_large_rows<false><<<dim3(gx, rows - 1), 256, 0, st>>>(*T, jobs, primes, m64, iL0, iL1, qg, qg_stride_words,
                                                                    k00, m32, 1, nullptr, 0);
            *nlaunch = 2;
        }
        return cudaGetLastError();
    }
    const bool pre = k00 != nullptr && m32 != nullptr && nslots > LS_GROUP; // one grid row: nothing to share
    if (pre) k_large_first<<<gx, 256, 0, st>>>(jobs, primes, m64, iL0, iL1, k00);
    *nlaunch = pre ? 2 : 1;
    k_large_strike<<<dim3(gx, (nslots + LS_GROUP - 1) / LS_GROUP), 256, 0, st>>>(
        jobs, nslots, primes, m64, iL0, iL1, qg, qg_stride_words, pre ? k00 : nullptr, pre ? m32 : nullptr);
    return cudaGetLastError();
}
cudaError_t launch_large_batch(const SegJob* jobs, const LargeBatchTab& T, const uint32_t* primes, const uint64_t* m64,
                               uint64_t i0, uint64_t i1, uint32_t* qg, uint64_t qg_stride_words, cudaStream_t st) {
    if (i1 <= i0 || !T.n) return cudaSuccess;
    const unsigned gx = (unsigned)std::min<uint64_t>((i1 - i0 + 255) / 256, 148ull * 16);
    k_large_batch<<<gx, 256, 0, st>>>(jobs, T, primes, m64, i0, i1, qg, qg_stride_words);
    return cudaGetLastError();
}
cudaError_t launch_large_m32(const uint64_t* m64, uint64_t iL0, uint64_t iL1, uint32_t* m32, cudaStream_t st) {
    if (iL1 <= iL0) return cudaSuccess;
    const unsigned gx = (unsigned)std::min<uint64_t>((iL1 - iL0 + 255) / 256, 148ull * 16);
    k_large_m32<<<gx, 256, 0, st>>>(m64, iL0, iL1, m32);
    return cudaGetLastError();
}
cudaError_t launch_mask_fill(const MaskArgs& a, uint32_t max_qg_words, cudaStream_t st) {
    if (!a.nslots || a.iK1 <= a.iK0) return cudaSuccess;
    const dim3 grid((max_qg_words + MK_WORDS - 1) / MK_WORDS, a.nslots);
    k_mask_fill<<<grid, MK_THREADS, MK_SMEM, st>>>(a);
    return cudaGetLastError();
}
cudaError_t launch_verify_blocks(const VerifyArgs& a, int grid, cudaStream_t st) {
    if (a.nslots > MAX_SLOTS) return cudaErrorInvalidValue; // s_jobs holds MAX_SLOTS
    // the sieve/check split follows the sieve's share of the work, which
    // grows with the number of tile primes (a.sw, chosen by the host)
    if (a.sw == WS_SW_HEAVY) {
        if (a.pmin_out) k_verify_ws<true, WS_SW_HEAVY><<<grid, WS_THREADS, WS_SMEM, st>>>(a);
        else k_verify_ws<false, WS_SW_HEAVY><<<grid, WS_THREADS, WS_SMEM, st>>>(a);
    } else if (a.sw == WS_SW_MASK) {
        if (a.pmin_out) k_verify_ws<true, WS_SW_MASK><<<grid, WS_THREADS, WS_SMEM, st>>>(a);
        else k_verify_ws<false, WS_SW_MASK><<<grid, WS_THREADS, WS_SMEM, st>>>(a);
    } else {
        if (a.pmin_out) k_verify_ws<true, WS_SW_LIGHT><<<grid, WS_THREADS, WS_SMEM, st>>>(a);
        else k_verify_ws<false, WS_SW_LIGHT><<<grid, WS_THREADS, WS_SMEM, st>>>(a);
    }
    return cudaGetLastError();
}
template <bool PMIN, int SW>
static cudaError_t launch_pair_t(const VerifyArgs& a, int grid, cudaStream_t st) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(WS_THREADS);
    cfg.dynamicSmemBytes = WS_SMEM;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_verify_pair<PMIN, SW>, a);
}
cudaError_t launch_verify_pairs(const VerifyArgs& a, int grid, cudaStream_t st) {
    if (a.nslots > MAX_SLOTS) return cudaErrorInvalidValue;
    grid &= ~1;
    if (grid < 2) grid = 2;
    cudaError_t e;
    if (a.sw == WS_SW_HEAVY) e = a.pmin_out ? launch_pair_t<true, WS_SW_HEAVY>(a, grid, st) : launch_pair_t<false, WS_SW_HEAVY>(a, grid, st);
    else if (a.sw == WS_SW_MASK) e = a.pmin_out ? launch_pair_t<true, WS_SW_MASK>(a, grid, st) : launch_pair_t<false, WS_SW_MASK>(a, grid, st);
    else e = a.pmin_out ? launch_pair_t<true, WS_SW_LIGHT>(a, grid, st) : launch_pair_t<false, WS_SW_LIGHT>(a, grid, st);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}
// per device, only when pair mode is used (lazy module loading keeps the
// cluster kernels out of every other open)
int pair_setup() {
    return (cudaFuncSetAttribute(k_verify_pair<false, WS_SW_LIGHT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)WS_SMEM) != cudaSuccess ||
            cudaFuncSetAttribute(k_verify_pair<true, WS_SW_LIGHT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)WS_SMEM) != cudaSuccess ||
            cudaFuncSetAttribute(k_verify_pair<false, WS_SW_HEAVY>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)WS_SMEM) != cudaSuccess ||
            cudaFuncSetAttribute(k_verify_pair<true, WS_SW_HEAVY>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)WS_SMEM) != cudaSuccess ||
            cudaFuncSetAttribute(k_verify_pair<false, WS_SW_MASK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)WS_SMEM) != cudaSuccess ||
            cudaFuncSetAttribute(k_verify_pair<true, WS_SW_MASK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)WS_SMEM) != cudaSuccess)
               ? 1 : 0;
}
int pair_clusters_resident(int* clusters) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(296);
    cfg.blockDim = dim3(WS_THREADS);
    cfg.dynamicSmemBytes = WS_SMEM;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaOccupancyMaxActiveClusters(clusters, k_verify_pair<false, WS_SW_HEAVY>, &cfg) == cudaSuccess ? 0 : 1;
}
cudaError_t launch_stragglers(const SegJob* jobs, const StragEntry* list, const unsigned int* list_count,
                              uint32_t list_cap, uint64_t p_small, StragResult* res, uint64_t* pmin_out,
                              int grid, cudaStream_t st) {
    k_stragglers<<<grid, 128, 0, st>>>(jobs, list, list_count, list_cap, p_small, res, pmin_out);
    return cudaGetLastError();
}
cudaError_t launch_finalize(const SegJob* jobs, uint32_t nslots, const SlotAcc* acc, const StragEntry* list,
                            const unsigned int* list_count, uint32_t list_cap, const StragResult* res,
                            DevRecord* out, cudaStream_t st) {
    k_finalize<<<1, 32, 0, st>>>(jobs, nslots, acc, list, list_count, list_cap, res, out);
    return cudaGetLastError();
}
cudaError_t launch_phase2_one(uint64_t n, uint64_t* out, cudaStream_t st) {
    k_phase2_one<<<1, 128, 0, st>>>(n, out);
    return cudaGetLastError();
}
cudaError_t launch_is_prime_batch(const uint64_t* v, uint8_t* out, uint64_t n, cudaStream_t st) {
    if (!n) return cudaSuccess;
    unsigned grid = (unsigned)std::min<uint64_t>((n + 255) / 256, 148ull * 8);
    k_is_prime_batch<<<grid, 256, 0, st>>>(v, out, n);
    return cudaGetLastError();
}
int verify_occupancy(int* blocks_per_sm) {
    // per-device function attributes: call after cudaSetDevice
    if (cudaFuncSetAttribute(k_sieve_interval, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SIEVE_SMEM) !=
        cudaSuccess)
        return 1;
    if (cudaFuncSetAttribute(k_mask_fill, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)MK_SMEM) != cudaSuccess)
        return 1;
    if (cudaFuncSetAttribute(k_verify_ws<false, WS_SW_LIGHT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)WS_SMEM) != cudaSuccess ||
        cudaFuncSetAttribute(k_verify_ws<true, WS_SW_LIGHT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)WS_SMEM) != cudaSuccess ||
        cudaFuncSetAttribute(k_verify_ws<false, WS_SW_HEAVY>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)WS_SMEM) != cudaSuccess ||
        cudaFuncSetAttribute(k_verify_ws<true, WS_SW_HEAVY>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)WS_SMEM) != cudaSuccess)
        return 1;
    if (cudaFuncSetAttribute(k_verify_ws<false, WS_SW_MASK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)WS_SMEM) != cudaSuccess ||
        cudaFuncSetAttribute(k_verify_ws<true, WS_SW_MASK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)WS_SMEM) != cudaSuccess)
        return 1;
    int o1 = 0, o2 = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, k_verify_ws<false, WS_SW_LIGHT>, WS_THREADS, WS_SMEM) !=
            cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, k_verify_ws<false, WS_SW_HEAVY>, WS_THREADS, WS_SMEM) !=
            cudaSuccess)
        return 1;
    *blocks_per_sm = o1 < o2 ? o1 : o2;
    return 0;
}

} // namespace gbk
