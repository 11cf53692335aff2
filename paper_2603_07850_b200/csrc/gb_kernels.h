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
    const uint32_t* primes;
    uint32_t iA0, iA1, iB1;       // tile prime index ranges
    uint32_t iW1;                 // first tile prime >= W (strikes a block at most once)
    uint32_t np;                  // pmc row length (iB1 - iA0)
    const uint4* pmc;             // nslots * np {p, floor(2^32/p), p - 1 - c0, c0}
    const uint16_t* wsplit;       // [SPLIT_WARPS][32] warp-cooperative row indices (0xFFFF = none)
    const uint32_t* qg;           // large-prime bitmask (nullptr = none)
    uint64_t qg_stride_words;
    const uint32_t* gpat;
    const uint64_t* pmr;
    uint64_t p_small;
    uint64_t inject;
    unsigned int* block_counter;
    SlotAcc* acc;
    StragEntry* list;
    unsigned int* list_count;
    uint32_t list_cap;
    uint64_t* pmin_out;           // optional per-even output (single slot)
};

// dynamic shared memory of the tile kernels
// k_verify_blocks dynamic smem: [tile | 4 pad words][patterns][pmr (8-B aligned)]
constexpr uint32_t VERIFY_PAT_OFF = TILE_WORDS + 4;
constexpr uint32_t VERIFY_PMR_OFF = (VERIFY_PAT_OFF + PAT_WORDS + 3) & ~3u; // 16-B aligned, in words
constexpr size_t VERIFY_SMEM = (size_t)VERIFY_PMR_OFF * 4 + NWIN * 8;
constexpr size_t SIEVE_SMEM = (TILE_WORDS + 1 + PAT_WORDS) * 4;
// k_verify_ws dynamic smem: [tile 0 | 4 pad][tile 1 | 4 pad][patterns][pmr]
constexpr uint32_t WS_PAT_OFF = 2 * (TILE_WORDS + 4);
constexpr uint32_t WS_PMR_OFF = (WS_PAT_OFF + PAT_WORDS + 3) & ~3u;
constexpr size_t WS_SMEM = (size_t)WS_PMR_OFF * 4 + NWIN * 8;

// ---- launchers (gb_kernels.cu); all asynchronous on `st`
cudaError_t launch_init_tables(uint32_t* pat, uint64_t* pmr, uint64_t p_small, cudaStream_t st);
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
                                uint64_t iL0, uint64_t iL1, uint32_t* qg, uint64_t qg_stride_words, cudaStream_t st);
cudaError_t launch_verify_blocks(const VerifyArgs& a, int grid, cudaStream_t st);
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
constexpr int SMEM_PEAK_THREADS = 512; // k_smem_peak: 2 CTAs x 512 threads per SM

} // namespace gbk
