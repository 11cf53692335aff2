// gb_kernels.h -- kernel-side types and host launchers (internal to the
// shared library; the public boundary is include/goldbach_b200.h).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "gb_device.cuh"
#include "../../include/goldbach_b200.h"

namespace gbk {

// Device-side segment record (finalize output), copied to gb_seg_record.
struct DevRecord {
    uint64_t a, b, evens;
    uint64_t unverified, phase2;
    uint64_t pmin_sum, pmin_hash;
    uint64_t max_p, max_n;
    uint64_t n_ce;
    uint64_t ce[GB_REC_MAX_CE];
    uint64_t overflow;
};

struct VerifyArgs {
    const SegJob* jobs;
    uint32_t nslots;
    uint32_t total_blocks;
    const uint32_t* primes;       // all base primes (low-window fix-up)
    uint64_t n_primes;
    uint64_t sbound;              // max(sqrt bound, 47): windows starting at or below need the fix-up
    uint32_t iA0, iA1, iB1;       // tile prime index ranges
    uint32_t iQ1, iH1;            // first tile primes >= M6/4, >= M6/2 (at most 4 / 2 strikes per array)
    uint32_t iW1;                 // first tile prime >= M6 (strikes an array at most once)
    uint32_t np;                  // pmc row length (iB1 - iA0)
    uint32_t sw;                  // sieve warps of the kernel split (WS_SW_LIGHT / WS_SW_HEAVY)
    const uint4* pmc;             // nslots * np {p, floor(2^32/p), p - 1 - k0, 4 6^-1 mod p}
    const uint16_t* wsplit;       // [SPLIT_WARPS][32] warp-cooperative row indices (0xFFFF = none)
    const uint32_t* qg;           // large-prime wheel-6 bitmask (nullptr = none)
    uint64_t qg_stride_words;
    const uint32_t* gpat6;        // wheel-6 presieve patterns
    const uint64_t* masks6;       // 3 x NWIN6 deep-window prime masks
    uint64_t p_small;
    uint64_t inject;
    unsigned int* block_counter;
    SlotAcc* acc;
    StragEntry* list;
    unsigned int* list_count;
    uint32_t list_cap;
    uint64_t* pmin_out;           // optional per-even output (single slot)
    uint32_t* tile_out;           // parity hook: the sieved tile of flat block tile_fb (A then B, 2 M6W words)
    uint32_t tile_fb;
    uint32_t total_pairs;         // k_verify_pair: block pairs of the batch (2-CTA clusters)
    unsigned int* pair_counter;
    // rows stop at iK0: tile primes from iK0 on are struck into qg by
    // k_mask_fill (iK0 = iB1 when the mask fill is off)
    uint32_t iK0;
};

// Slot layout of one batch on a common wheel axis (k_large_batch): slot s's
// window is cells [d[s], d[s] + its qg_words * 32) of q = Q_0 + 6k.  Valid only
// for ascending, near slots whose windows overlap at most their neighbours
// (host-checked per batch); unused entries d = ~0.
struct LargeBatchTab {
    uint32_t d[MAX_SLOTS];
    uint32_t qw[MAX_SLOTS]; // qg_words of each slot
    uint32_t qm[MAX_SLOTS][2]; // (slot origin + 4 arr) mod 5005, arr 0 = A, 1 = B
    uint32_t qm2[MAX_SLOTS][2]; // the same mod 7429
    uint32_t cop;  // k_large_rows: skip strikes of multiples of 5, 7, 11, 13 (1), and of 17, 19, 23 (2); 0 = none
    uint32_t n;    // slots
    uint32_t span; // max over s of d[s] + cells of slot s
};

struct MaskArgs {
    const SegJob* jobs;           // qg_words per slot
    uint32_t nslots;
    const uint4* pmc;             // rows of [iA0, iA0 + np) per slot
    uint32_t np, iA0;
    uint32_t iK0, iK1;            // mask primes (row indices are i - iA0)
    uint32_t* qg;
    uint64_t qg_stride_words;
};

// dynamic shared memory of the tile kernels
constexpr size_t SIEVE_SMEM = (TILE_WORDS + 1 + PAT_WORDS) * 4;
// k_verify_ws dynamic smem: [tile 0][tile 1] (wheel-6, TILE6_WORDS each)[patterns][masks6]
constexpr uint32_t WS_PAT_OFF = 2 * TILE6_WORDS;
constexpr uint32_t WS_MASK_OFF = (WS_PAT_OFF + PAT6_WORDS + 3) & ~3u;
constexpr size_t WS_SMEM = (size_t)WS_MASK_OFF * 4 + 3 * NWIN6 * 8;

// ---- launchers (gb_kernels.cu); all asynchronous on `st`
cudaError_t launch_init_tables(uint32_t* pat, uint32_t* pat6, uint64_t* masks6, uint64_t p_small, cudaStream_t st);
cudaError_t launch_seed_primes(uint32_t lim, uint32_t* out, uint32_t* count, cudaStream_t st);
cudaError_t launch_sieve_interval(uint64_t lo, uint64_t n_cells, const uint32_t* primes, uint32_t iA0,
                                  uint32_t iA1, uint32_t iB1, const uint32_t* pat, uint32_t* out,
                                  int grid, cudaStream_t st);
cudaError_t launch_count_words(const uint32_t* bits, uint64_t n_words, uint32_t chunk, uint32_t* counts,
                               uint64_t n_chunks, cudaStream_t st);
cudaError_t launch_scan(const uint32_t* counts, uint64_t n, uint64_t* offsets, uint64_t* total,
                        cudaStream_t st);
cudaError_t launch_compact(const uint32_t* bits, uint64_t n_words, uint32_t chunk, const uint64_t* offsets,
                           uint64_t lo, uint32_t* primes, uint64_t n_chunks, cudaStream_t st);
cudaError_t launch_prime_magic64(const uint32_t* primes, uint64_t n, uint64_t* m64, cudaStream_t st);
cudaError_t launch_segment_offsets(const SegJob* jobs, uint32_t nslots, const uint32_t* primes,
                                   const uint64_t* m64, uint32_t iA0, uint32_t np, uint4* pmc, cudaStream_t st);
cudaError_t launch_large_strike(const SegJob* jobs, uint32_t nslots, const uint32_t* primes, const uint64_t* m64,
                                uint64_t iL0, uint64_t iL1, uint32_t* qg, uint64_t qg_stride_words, uint32_t* k00,
                                const uint32_t* m32, const LargeBatchTab* T, const uint32_t* k00_prev, uint32_t dd,
                                int* nlaunch, cudaStream_t st);
cudaError_t launch_large_batch(const SegJob* jobs, const LargeBatchTab& T, const uint32_t* primes, const uint64_t* m64,
                               uint64_t i0, uint64_t i1, uint32_t* qg, uint64_t qg_stride_words, cudaStream_t st);
cudaError_t launch_large_m32(const uint64_t* m64, uint64_t iL0, uint64_t iL1, uint32_t* m32, cudaStream_t st);
cudaError_t launch_mask_fill(const MaskArgs& a, uint32_t max_qg_words, cudaStream_t st);
cudaError_t launch_verify_blocks(const VerifyArgs& a, int grid, cudaStream_t st);
// paired variant: 2-CTA clusters, each single-strike row visited once per
// block pair (grid rounded down to whole clusters)
cudaError_t launch_verify_pairs(const VerifyArgs& a, int grid, cudaStream_t st);
int pair_clusters_resident(int* clusters);
int pair_setup(); // cluster kernels' shared-memory attribute (pair mode only)
cudaError_t launch_stragglers(const SegJob* jobs, const StragEntry* list, const unsigned int* list_count,
                              uint32_t list_cap, uint64_t p_small, StragResult* res, uint64_t* pmin_out,
                              int grid, cudaStream_t st);
cudaError_t launch_finalize(const SegJob* jobs, uint32_t nslots, const SlotAcc* acc, const StragEntry* list,
                            const unsigned int* list_count, uint32_t list_cap, const StragResult* res,
                            DevRecord* out, cudaStream_t st);
cudaError_t launch_phase2_one(uint64_t n, uint64_t* out, cudaStream_t st);
cudaError_t launch_is_prime_batch(const uint64_t* v, uint8_t* out, uint64_t n, cudaStream_t st);
cudaError_t launch_smem_peak(uint32_t iters, uint32_t* sink, int grid, cudaStream_t st);
int verify_occupancy(int* blocks_per_sm);
int debug_stats(unsigned long long* out, int reset); // GB_STATS builds only (returns 2 otherwise)
constexpr int SMEM_PEAK_THREADS = 512; // k_smem_peak: 2 CTAs x 512 threads per SM

} // namespace gbk
