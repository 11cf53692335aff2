/*
 * goldbach_b200.h -- C-ABI drop-in boundary of the B200 Goldbach verifier.
 *
 * The reference (arXiv 2603.07850, /root/reference/proj) verifies one
 * segment of even numbers per call to
 *
 *     SegmentReport verify_segment(const SegmentJob&, const VerifyContext&);
 *                                                  (proj/include/goldbach/verifier.hpp:116-118)
 *
 * implemented on the CPU as sieve_range_for -> tiled_sieve_segment ->
 * phase1_verify -> count_unverified -> phase2_resolve
 * (proj/src/verifier.cpp:167-206).  This header is the replacement's
 * boundary: plain pointers and integers, status codes instead of
 * exceptions, no C++ or torch types.  The C++ host layer
 * (paper_2603_07850_b200/csrc/host, same headers as proj/include/goldbach)
 * is the only production caller; it maps non-zero status codes back to the
 * reference exception taxonomy (proj/include/goldbach/errors.hpp:9-22):
 *   GB_ERR_PARAM    -> ParamError
 *   GB_ERR_RESOURCE -> ResourceError
 *   GB_ERR_INTERNAL -> InternalError
 *   GB_ERR_CUDA     -> std::runtime_error (device failure)
 *
 * Threading: one gb_dev per GPU, driven by exactly one host thread at a
 * time (the run_workers worker bound to that GPU, proj/src/pool.cpp:90-120).
 * gb_dev has no internal locking.
 *
 * Every function returns 0 on success.  gb_last_error() returns the message
 * of the last failure on that handle (thread-local message when dev==NULL).
 */
#ifndef GOLDBACH_B200_H
#define GOLDBACH_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GB_OK 0
#define GB_ERR_PARAM 1
#define GB_ERR_RESOURCE 2
#define GB_ERR_INTERNAL 3
#define GB_ERR_CUDA 4

/* Counterexamples recorded per segment (ascending).  The count is exact;
 * only the first GB_REC_MAX_CE values are stored. */
#define GB_REC_MAX_CE 16

/*
 * Per-segment verification record: the reference SegmentReport
 * (proj/include/goldbach/verifier.hpp:107-114) plus the minimal-p checksum.
 *
 *   evens_checked      = evens in [a, b]                  (verifier.cpp:179)
 *   unverified_p1      = evens not certified by Phase 1,
 *                        inject_fail included              (verifier.cpp:181-186)
 *   phase2_resolved    = leftovers resolved by Phase 2    (verifier.cpp:193-199)
 *   max_p / max_n      = MinPrimeMax: max p_min, smallest n on ties
 *                                                          (verifier.hpp:53-66)
 *   pmin_sum           = sum of p over every MinPrimeMax::observe(p, n) call
 *                        made for the segment, mod 2^64
 *   pmin_hash          = sum of p * (n >> 1) over the same calls, mod 2^64
 *
 * The checksum definition is this repo's (the reference exposes p_min only
 * through phase1_verify(..., min_primes_out), verifier.hpp:74-79); with no
 * Phase 2 it equals SURVEY.md Appendix A's sum_pmin / pos_hash exactly.
 */
typedef struct gb_seg_record {
    uint64_t a, b;
    uint64_t evens_checked;
    uint64_t unverified_p1;
    uint64_t phase2_resolved;
    uint64_t pmin_sum;
    uint64_t pmin_hash;
    uint64_t max_p, max_n;
    uint64_t n_counterexamples;
    uint64_t counterexamples[GB_REC_MAX_CE];
    double elapsed_seconds; /* host-observed submit->complete time */
} gb_seg_record;

/*
 * Device/table parameters: the pieces of VerifyContext (verifier.hpp:96-105)
 * and Config (cli.hpp:18-31) that shape the device state.
 *   cover_limit : base primes are the odd primes <= s, s the minimal s with
 *                 s >= cover_limit / s (build_base_primes, sieve.cpp:44-70);
 *                 run() passes cfg.limit (cli.cpp:314).
 *   p_small     : Phase 1 partition primes are the odd primes <= p_small
 *                 (SmallPrimeTable, verifier.hpp:22-27); >= 3.
 *   phase2_limit, batch_size : accepted for drop-in compatibility; both are
 *                 result-invariant (verifier.cpp:137-142,
 *                 test_verifier.cpp:121-137) and unused by the device path.
 *   inject_fail : self-test hook (verifier.hpp:102-104); 0 = off.
 *   max_seg_evens : largest segment this handle will be asked to verify;
 *                 sizes the device buffers (0 = 2e8).
 */
typedef struct gb_params {
    uint64_t cover_limit;
    uint64_t p_small;
    uint64_t phase2_limit;
    uint64_t batch_size;
    uint64_t inject_fail;
    uint64_t max_seg_evens;
} gb_params;

typedef struct gb_dev gb_dev;

/* Library version string and the compiled device architecture. */
const char* gb_version(void);

/* Number of CUDA devices visible (0 if none / no driver). */
int gb_device_count(int* count);

/* Opens device `device`, builds the base primes (K1, on device) and the
 * resident Phase 1 tables.  Replaces the table builds in run()
 * (cli.cpp:312-314) for one GPU. */
int gb_open(int device, const gb_params* params, gb_dev** out);
int gb_close(gb_dev* dev);
const char* gb_last_error(const gb_dev* dev);

/* Re-targets an open handle to a new inject_fail value (VerifyContext is
 * otherwise immutable for the life of the handle). */
int gb_set_inject_fail(gb_dev* dev, uint64_t inject_fail);

/* Synchronous verify_segment (verifier.cpp:167-206) for evens [a, b]:
 * a, b even, 4 <= a <= b (check_job, verifier.cpp:15-20), b below the
 * handle's cover limit ceiling.  Writes one record. */
int gb_verify_segment(gb_dev* dev, uint64_t a, uint64_t b, gb_seg_record* out);

/* Asynchronous form used by the per-GPU worker to keep the device busy:
 * at most gb_max_inflight() segments may be outstanding; gb_wait returns
 * them in submission order with the caller's tag. */
int gb_max_inflight(const gb_dev* dev, int* depth);
int gb_submit_segment(gb_dev* dev, uint64_t a, uint64_t b, uint64_t tag);
int gb_wait_segment(gb_dev* dev, gb_seg_record* out, uint64_t* tag);

/* Base-prime table built on the device (K1): sqrt_bound and count; copies
 * up to `cap` primes into `out` when out != NULL.  Parity hook for
 * build_base_primes (sieve.cpp:44-70). */
int gb_base_primes(gb_dev* dev, uint64_t* sqrt_bound, uint64_t* count,
                   uint32_t* out, uint64_t cap);

/* Odd primes <= limit (limit < 2^32) sieved on the device; copies up to
 * cap into out when out != NULL.  Backs simple_sieve / SmallPrimeTable /
 * Phase2Table::build of the C++ API (sieve.cpp:22-42). */
int gb_primes_upto(gb_dev* dev, uint64_t limit, uint32_t* out, uint64_t cap,
                   uint64_t* count);

/* Device sieve of the odd interval [lo, hi] (lo, hi odd, lo <= hi):
 * writes ((hi-lo)/2 + 64) / 64 words, bit i <-> lo + 2i, LSB-first, slack
 * bits zero: the OddBitset layout of tiled_sieve_segment (sieve.cpp:91-156,
 * oddbits.hpp:14-97).  Requires hi within the handle's cover limit. */
int gb_sieve_interval(gb_dev* dev, uint64_t lo, uint64_t hi, uint64_t* words,
                      uint64_t n_words);

/* Per-even Phase 1 minimal primes for [a, b] exactly as
 * phase1_verify(..., min_primes_out) (verifier.cpp:45-104): p_min(n), or 0
 * when Phase 1 does not certify n.  out has (b-a)/2+1 entries. */
int gb_phase1_pmin(gb_dev* dev, uint64_t a, uint64_t b, uint64_t* out,
                   uint64_t n_out);

/* Device deterministic Miller-Rabin (is_prime_u64, primality.cpp:32-52)
 * over a host array; parity hook for K4. */
int gb_is_prime_batch(gb_dev* dev, const uint64_t* values, uint8_t* out,
                      uint64_t count);

/* Parity hook for the fused kernel's own sieve (K2): runs [a, b] (one piece)
 * and copies the wheel-6 tile of block `block` right after its sieve, before
 * the check reads it.  *words_per_array = W (the tile's words per class
 * array; out_words == NULL only queries it).  out_words[0 .. W-1] = array A
 * (bit k of word w <-> q = origin + 6 (32 w + k)), out_words[W .. 2W-1] =
 * array B (q = origin + 4 + 6 (32 w + k)), cap_words >= 2W; *origin = the
 * block's window origin Q_b (1 mod 6, negative near the start of the number
 * line).  Bit set <=> q prime, for every q <= the handle's cover limit.  Not
 * part of the reference interface; below 2^63 only. */
int gb_debug_tile(gb_dev* dev, uint64_t a, uint64_t b, uint32_t block, uint32_t* out_words,
                  uint64_t cap_words, uint32_t* words_per_array, int64_t* origin);

/* Device Phase 2 resolver (phase2_resolve, verifier.cpp:129-165) for one
 * even n >= 4 with the handle's p_small: *p = minimal prime p (0 when none,
 * i.e. a counterexample). */
int gb_phase2_resolve(gb_dev* dev, uint64_t n, uint64_t* p);

/* Mask fill of the large tile primes (k_mask_fill: every base prime from
 * the threshold up to 2^22 struck once per 3-block range of a piece into
 * the piece's large-prime bitmask, instead of visited by every block --
 * the reference's sparse-prime hit list, sieve.cpp:109-126, in bitmask
 * form).  enabled = 0 puts those primes back on the per-block row path
 * (A/B timing; results are identical).  No segments may be pending.  Not
 * part of the reference interface. */
int gb_set_bucket(gb_dev* dev, int enabled);

/* Mask-fill plan: [0] active, [1] smallest mask prime, [2] mask primes,
 * [3] cells per fill range, [4] primes above 2^22 (k_large_strike);
 * [5..7] zero. */
int gb_bucket_info(const gb_dev* dev, uint64_t* out8);

/* Kernel launches issued by this handle since open (bench evidence). */
int gb_launch_count(const gb_dev* dev, uint64_t* launches);

/* Device time (ms) spent in each kernel family since the last reset,
 * measured with CUDA events on the handle's streams: [0]=segment sieve+check
 * (K2/K3 fused), [1]=pre-kernels (row offsets, mask fill, large-prime
 * strike), [2]=stragglers/Phase 2, [3]=other. */
int gb_kernel_times(gb_dev* dev, double* ms4, uint64_t* launches4, int reset);

/* Debug counters of the fused kernel, process-wide (builds with
 * -DGB_STATS only; GB_ERR_PARAM otherwise): [0] evens checked per even on
 * the generic path, [1] deep evens resolved in place (queue overflow),
 * [2] deep evens queued, [3] deep rounds, [4] straggler entries, [5] fast
 * blocks, [6] generic blocks.  Not part of the reference interface. */
int gb_debug_stats(uint64_t* out8, int reset);

/* Per-launch event timing: 0 off, 1 on, 2 on with every batch serialised on
 * one stream (so an event pair brackets exactly one kernel's execution;
 * used for the roofline pass of bench.py).  No segments may be pending. */
int gb_set_timing(gb_dev* dev, int enabled);

/* Host<->device bytes moved by segment traffic since open (job descriptors
 * in, records out). */
int gb_io_bytes(const gb_dev* dev, uint64_t* h2d, uint64_t* d2h);

/* Writes 256 MiB of scratch (> the 126 MB L2) and synchronises: evicts L2
 * between timed iterations. */
int gb_flush_l2(gb_dev* dev);

/* cudaDeviceSynchronize on the handle's device. */
int gb_synchronize(gb_dev* dev);

/* Device-clock interval timer (CUDA events): op 0 drains the device and
 * records the start event; op 1 drains the device, records the stop event
 * and writes the elapsed milliseconds to *ms.  Used by bench.py. */
int gb_device_timer(gb_dev* dev, int op, double* ms);

/* Measured shared-memory load bandwidth of the device in bytes/s
 * (conflict-free 128-bit loads from 2 CTAs x 512 threads on every SM):
 * the roofline denominator of the fused sieve+check kernel. */
int gb_smem_peak(gb_dev* dev, double* bytes_per_s);

#ifdef __cplusplus
}
#endif

#endif /* GOLDBACH_B200_H */
