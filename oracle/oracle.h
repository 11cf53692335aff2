/*
 * oracle.h -- CPU restatement of the reference verification path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker for the B200 path:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it.  The product (paper_2603_07850_b200) never links or calls it.
 *
 * Every function restates one reference function; the citation is the
 * file:line under /root/reference/proj it follows.  Parity is pinned two
 * ways: against the reference's own known-answer
 * tests (tests/test_oracle_*.py) and against golden vectors produced by
 * the reference itself, compiled here into oracle/_ref (oracle/make_goldens.py).
 */
#ifndef GB_ORACLE_H
#define GB_ORACLE_H

#include <stdint.h>
#include "../include/goldbach_b200.h" /* gb_seg_record */

#ifdef __cplusplus
extern "C" {
#endif

/* primality.hpp:16-19 / primality.cpp:5-15 / primality.cpp:32-52 */
uint64_t or_modmul(uint64_t a, uint64_t b, uint64_t m);
uint64_t or_modpow(uint64_t a, uint64_t e, uint64_t m);
int or_is_prime_u64(uint64_t n);

/* sieve.cpp:22-42: primes <= limit including 2; returns count, fills out
 * when out != NULL and cap is large enough (else -1). */
int64_t or_simple_sieve(uint64_t limit, uint64_t* out, uint64_t cap);

/* sieve.cpp:48-52: minimal s with s >= cover / s */
uint64_t or_sqrt_bound(uint64_t cover_limit);

/* sieve.cpp:44-70: odd primes <= sqrt_bound(cover); returns count. */
int64_t or_build_base_primes(uint64_t cover_limit, uint32_t* out, uint64_t cap,
                             uint64_t* sqrt_bound);

/* sieve.cpp:72-89: 1 and *idx set, or 0 (nullopt). -1 on ParamError. */
int or_first_tile_index(uint64_t p, uint64_t tile_lo, uint64_t seg_hi,
                        uint64_t* idx);

/* sieve.cpp:91-156: OddBitset words for odd [lo, hi] using the given base
 * primes and tile size; returns 0, or -1 on ParamError. words must hold
 * ((hi-lo)/2+64)/64 entries. */
int or_tiled_sieve_segment(uint64_t lo, uint64_t hi, const uint32_t* base,
                           uint64_t n_base, uint64_t sqrt_bound,
                           uint64_t odds_per_tile, uint64_t* words);

/* verifier.cpp:35-43; returns -1 on ParamError (check_job :15-20). */
int or_sieve_range_for(uint64_t a, uint64_t b, uint64_t p_small, uint64_t* lo,
                       uint64_t* hi);

/* verifier.cpp:45-104 with min_primes_out: p_min per even (0 = not
 * certified).  qbits/q_lo/q_hi is an OddBitset covering sieve_range_for.
 * small = odd primes <= p_small ascending (the table without the leading 2).
 * Returns 0, -1 ParamError, -2 InternalError (coverage). */
int or_phase1_pmin(uint64_t a, uint64_t b, const uint64_t* small_odd,
                   uint64_t n_small_odd, const uint64_t* qbits, uint64_t q_lo,
                   uint64_t q_hi, uint64_t* pmin_out);

/* verifier.cpp:129-165 with the Phase 2 table disabled (result-invariant:
 * both lookups are exact, verifier.cpp:137-142).  Returns p or 0 when no
 * partition exists (counterexample). */
uint64_t or_phase2_resolve(uint64_t n, uint64_t p_small);

/* verifier.cpp:167-206: the full per-segment report plus this repo's
 * checksum (sum / pos-hash over every MinPrimeMax::observe).  Builds its
 * own tables: base primes for cover_limit, small primes <= p_small.
 * Returns 0, -1 ParamError, -2 InternalError. */
int or_verify_segment(uint64_t a, uint64_t b, uint64_t cover_limit,
                      uint64_t p_small, uint64_t inject_fail,
                      gb_seg_record* rec);

/* Same as or_verify_segment but reusing caller tables (for drivers that run
 * many segments).  base: odd primes <= sqrt_bound; small_odd: odd primes
 * <= p_small. */
int or_verify_segment_tables(uint64_t a, uint64_t b, const uint32_t* base,
                             uint64_t n_base, uint64_t sqrt_bound,
                             const uint64_t* small_odd, uint64_t n_small_odd,
                             uint64_t p_small, uint64_t inject_fail,
                             gb_seg_record* rec);

/* Multi-threaded range driver (WorkPool + run_workers semantics,
 * pool.cpp:24-31 / 70-175) used as the CPU baseline when the compiled
 * reference is unavailable: returns the merged record over [start, limit]
 * with segments of seg_size evens, `threads` workers. */
int or_verify_range(uint64_t start, uint64_t limit, uint64_t seg_size,
                    uint64_t cover_limit, uint64_t p_small, int threads,
                    gb_seg_record* total, uint64_t* segments);

#ifdef __cplusplus
}
#endif
#endif
