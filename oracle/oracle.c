/*
 * oracle.c -- CPU restatement of the reference verification path
 * (arXiv 2603.07850, /root/reference/proj/src).
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Plain C11, no GMP: the
 * reference's GMP cross-checks (tests/oracle.cpp:8-40) are replaced by the
 * deterministic 12-witness Miller-Rabin it validates (primality.cpp:32-52)
 * plus trial division in the tests.
 */
#include "oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

/* primality.hpp:16-19 */
uint64_t or_modmul(uint64_t a, uint64_t b, uint64_t m) {
    return (uint64_t)((u128)a * b % m);
}

/* primality.cpp:5-15 */
uint64_t or_modpow(uint64_t a, uint64_t e, uint64_t m) {
    uint64_t result = 1 % m;
    a %= m;
    while (e) {
        if (e & 1) result = or_modmul(result, a, m);
        a = or_modmul(a, a, m);
        e >>= 1;
    }
    return result;
}

static const uint32_t kWitnesses[12] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};

/* primality.cpp:20-28 */
static int witness_passes(uint64_t n, uint64_t a, uint64_t d, int s) {
    uint64_t x = or_modpow(a, d, n);
    if (x == 1 || x == n - 1) return 1;
    for (int r = 1; r < s; ++r) {
        x = or_modmul(x, x, n);
        if (x == n - 1) return 1;
    }
    return 0;
}

/* primality.cpp:32-52 */
int or_is_prime_u64(uint64_t n) {
    if (n < 41) {
        for (int i = 0; i < 12; ++i)
            if (n == kWitnesses[i]) return 1;
        return 0;
    }
    for (int i = 0; i < 12; ++i)
        if (n % kWitnesses[i] == 0) return 0;
    uint64_t d = n - 1;
    int s = 0;
    while ((d & 1) == 0) {
        d >>= 1;
        ++s;
    }
    for (int i = 0; i < 12; ++i)
        if (!witness_passes(n, kWitnesses[i], d, s)) return 0;
    return 1;
}

/* sieve.cpp:22-42 (the mem-cap ResourceError at :24-28 is the caller's) */
int64_t or_simple_sieve(uint64_t limit, uint64_t* out, uint64_t cap) {
    if (limit < 2) return -1;
    uint8_t* composite = (uint8_t*)calloc(limit + 1, 1);
    if (!composite) return -1;
    for (uint64_t i = 3; i <= limit / i; i += 2) {
        if (composite[i]) continue;
        for (uint64_t j = i * i; j <= limit; j += 2 * i) composite[j] = 1;
    }
    int64_t count = 0;
    if (out && cap > 0) out[0] = 2;
    count = 1;
    for (uint64_t i = 3; i <= limit; i += 2)
        if (!composite[i]) {
            if (out && (uint64_t)count < cap) out[count] = i;
            ++count;
        }
    free(composite);
    if (out && (uint64_t)count > cap) return -1;
    return count;
}

/* sieve.cpp:48-52 */
uint64_t or_sqrt_bound(uint64_t cover_limit) {
    uint64_t s = (uint64_t)sqrtl((long double)cover_limit);
    if (s == 0) s = 1;
    while (s > 1 && (s - 1) >= cover_limit / (s - 1)) --s;
    while (s < cover_limit / s) ++s;
    return s;
}

/* sieve.cpp:44-70 */
int64_t or_build_base_primes(uint64_t cover_limit, uint32_t* out, uint64_t cap,
                             uint64_t* sqrt_bound) {
    if (cover_limit < 1) return -1;
    uint64_t s = or_sqrt_bound(cover_limit);
    if (sqrt_bound) *sqrt_bound = s;
    if (s < 3) return 0;
    uint64_t n_bits = (s - 3) / 2 + 1;
    uint64_t n_words = (n_bits + 63) / 64;
    uint64_t* flags = (uint64_t*)malloc(n_words * 8);
    if (!flags) return -1;
    memset(flags, 0xff, n_words * 8);
    for (uint64_t v = 3; v <= s / v; v += 2) {
        uint64_t i = (v - 3) >> 1;
        if (!((flags[i >> 6] >> (i & 63)) & 1)) continue;
        for (uint64_t m = v * v; m <= s; m += 2 * v) {
            uint64_t k = (m - 3) >> 1;
            flags[k >> 6] &= ~(1ULL << (k & 63));
        }
    }
    int64_t count = 0;
    for (uint64_t i = 0; i < n_bits; ++i)
        if ((flags[i >> 6] >> (i & 63)) & 1) {
            if (out && (uint64_t)count < cap) out[count] = (uint32_t)(3 + 2 * i);
            ++count;
        }
    free(flags);
    if (out && (uint64_t)count > cap) return -1;
    return count;
}

/* sieve.cpp:72-89 */
int or_first_tile_index(uint64_t p, uint64_t tile_lo, uint64_t seg_hi,
                        uint64_t* idx) {
    if (p < 3 || (p & 1) == 0) return -1;
    if ((tile_lo & 1) == 0 || (seg_hi & 1) == 0) return -1;
    uint64_t c = tile_lo / p;
    if (c * p < tile_lo) ++c;
    if (c < p) c = p;
    if ((c & 1) == 0) ++c;
    if (c > seg_hi / p) return 0;
    uint64_t m = p * c;
    *idx = (m - tile_lo) >> 1;
    return 1;
}

static int cmp_u64(const void* x, const void* y) {
    uint64_t a = *(const uint64_t*)x, b = *(const uint64_t*)y;
    return a < b ? -1 : a > b;
}

/* sieve.cpp:91-156 (stride primes carried across tiles :113-143, sparse
 * hits pre-sorted :126, 1 cleared :154) */
int or_tiled_sieve_segment(uint64_t lo, uint64_t hi, const uint32_t* base,
                           uint64_t n_base, uint64_t s,
                           uint64_t odds_per_tile, uint64_t* words) {
    if ((lo & 1) == 0 || (hi & 1) == 0) return -1;
    if (lo > hi) return -1;
    uint64_t t_bits = odds_per_tile;
    if (t_bits < 64 || (t_bits & (t_bits - 1)) != 0) return -1;
    if (s == 0 || s < hi / s) return -1;

    uint64_t span = hi - lo;
    uint64_t n_bits = (span >> 1) + 1;
    uint64_t n_words = (n_bits + 63) >> 6;

    uint64_t* stride_p = (uint64_t*)malloc((n_base + 1) * 8);
    uint64_t* stride_next = (uint64_t*)malloc((n_base + 1) * 8);
    uint64_t* sparse = (uint64_t*)malloc((n_base + 1) * 8);
    uint64_t n_stride = 0, n_sparse = 0;
    for (uint64_t k = 0; k < n_base; ++k) {
        uint64_t p = base[k];
        if (p > hi / p) break;
        uint64_t idx;
        if (or_first_tile_index(p, lo, hi, &idx) != 1) continue;
        if (2 * p <= span) {
            stride_p[n_stride] = p;
            stride_next[n_stride++] = idx;
        } else {
            sparse[n_sparse++] = idx;
        }
    }
    qsort(sparse, n_sparse, 8, cmp_u64);

    uint64_t* tile = (uint64_t*)malloc((t_bits / 64) * 8);
    uint64_t hit_at = 0;
    for (uint64_t t0 = 0; t0 < n_bits; t0 += t_bits) {
        uint64_t t1 = t0 + t_bits < n_bits ? t0 + t_bits : n_bits;
        memset(tile, 0xff, (t_bits / 64) * 8);
        for (uint64_t i = 0; i < n_stride; ++i) {
            uint64_t idx = stride_next[i], p = stride_p[i];
            while (idx < t1) {
                uint64_t r = idx - t0;
                tile[r >> 6] &= ~(1ULL << (r & 63));
                idx += p;
            }
            stride_next[i] = idx;
        }
        while (hit_at < n_sparse && sparse[hit_at] < t1) {
            uint64_t r = sparse[hit_at++] - t0;
            tile[r >> 6] &= ~(1ULL << (r & 63));
        }
        uint64_t nw = (t1 - t0 + 63) >> 6;
        memcpy(words + (t0 >> 6), tile, nw * 8);
    }
    if (n_bits & 63) words[n_words - 1] &= (1ULL << (n_bits & 63)) - 1; /* mask_tail */
    if (lo == 1) words[0] &= ~1ULL;
    free(tile);
    free(stride_p);
    free(stride_next);
    free(sparse);
    return 0;
}

/* verifier.cpp:15-20 */
static int check_job(uint64_t a, uint64_t b) {
    if ((a & 1) || (b & 1)) return -1;
    if (a < 4 || a > b) return -1;
    return 0;
}

/* verifier.cpp:35-43 */
int or_sieve_range_for(uint64_t a, uint64_t b, uint64_t p_small, uint64_t* lo,
                       uint64_t* hi) {
    if (check_job(a, b)) return -1;
    uint64_t l = a > p_small ? a - p_small : 0;
    if (l < 3) l = 3;
    if ((l & 1) == 0) ++l;
    uint64_t h = b - 3;
    if (h < l) h = l;
    *lo = l;
    *hi = h;
    return 0;
}

static inline int qtest(const uint64_t* qbits, uint64_t q_lo, uint64_t v) {
    uint64_t i = (v - q_lo) >> 1;
    return (qbits[i >> 6] >> (i & 63)) & 1;
}

/* verifier.cpp:45-104.  The batch_size chunking (:75-103) is
 * result-invariant (test_verifier.cpp:121-137): one ascending scan over the
 * odd small primes with early exit is the same computation. */
int or_phase1_pmin(uint64_t a, uint64_t b, const uint64_t* odd, uint64_t n_odd,
                   const uint64_t* qbits, uint64_t q_lo, uint64_t q_hi,
                   uint64_t* pmin_out) {
    if (check_job(a, b)) return -1;
    uint64_t p_small = 0;
    (void)p_small;
    uint64_t n_evens = ((b - a) >> 1) + 1;
    for (uint64_t i = 0; i < n_evens; ++i) {
        uint64_t n = a + 2 * i;
        pmin_out[i] = 0;
        if (n == 4) {
            pmin_out[i] = 2; /* verifier.cpp:92-95 */
            continue;
        }
        for (uint64_t k = 0; k < n_odd; ++k) {
            uint64_t p = odd[k];
            if (p > n - 3) break; /* verifier.cpp:81 */
            uint64_t q = n - p;
            if (q < q_lo || q > q_hi) return -2; /* coverage, verifier.cpp:55-57 */
            if (qtest(qbits, q_lo, q)) {
                pmin_out[i] = p;
                break;
            }
        }
    }
    return 0;
}

/* verifier.cpp:129-165 with phase2.limit < 2 (every q-test by MR). */
uint64_t or_phase2_resolve(uint64_t n, uint64_t p_small) {
    uint64_t half = n / 2;
    /* small primes ascending from 2 (:145-148) */
    if (2 <= half && or_is_prime_u64(n - 2)) return 2;
    for (uint64_t p = 3; p <= p_small; p += 2) {
        if (!or_is_prime_u64(p)) continue;
        if (p > half) return 0;
        if (or_is_prime_u64(n - p)) return p;
    }
    /* raw odd candidates past p_small (:162-163) */
    uint64_t from = p_small;
    for (uint64_t p = (from & 1) ? from + 2 : from + 1; p <= half; p += 2)
        if (or_is_prime_u64(p) && or_is_prime_u64(n - p)) return p;
    return 0;
}

/* MinPrimeMax::observe (verifier.hpp:57-62) + this repo's checksum. */
static void observe(gb_seg_record* r, uint64_t p, uint64_t n) {
    r->pmin_sum += p;
    r->pmin_hash += p * (n >> 1);
    if (p > r->max_p || (p == r->max_p && r->max_p != 0 && n < r->max_n)) {
        r->max_p = p;
        r->max_n = n;
    }
}

static void add_ce(gb_seg_record* r, uint64_t n) {
    if (r->n_counterexamples < GB_REC_MAX_CE) r->counterexamples[r->n_counterexamples] = n;
    r->n_counterexamples++;
}

/* verifier.cpp:167-206 */
int or_verify_segment_tables(uint64_t a, uint64_t b, const uint32_t* base,
                             uint64_t n_base, uint64_t s,
                             const uint64_t* odd, uint64_t n_odd,
                             uint64_t p_small, uint64_t inject_fail,
                             gb_seg_record* rec) {
    memset(rec, 0, sizeof(*rec));
    rec->a = a;
    rec->b = b;
    uint64_t lo, hi;
    if (or_sieve_range_for(a, b, p_small, &lo, &hi)) return -1;
    uint64_t n_bits = ((hi - lo) >> 1) + 1;
    uint64_t* qbits = (uint64_t*)calloc((n_bits + 63) / 64 + 1, 8);
    if (or_tiled_sieve_segment(lo, hi, base, n_base, s, 32768, qbits)) {
        free(qbits);
        return -1;
    }
    uint64_t n_evens = ((b - a) >> 1) + 1;
    uint64_t* pmin = (uint64_t*)malloc(n_evens * 8);
    int rc = or_phase1_pmin(a, b, odd, n_odd, qbits, lo, hi, pmin);
    free(qbits);
    if (rc) {
        free(pmin);
        return rc;
    }
    rec->evens_checked = n_evens;
    /* Phase 1 observations (phase1_verify's mark, verifier.cpp:78-81) */
    for (uint64_t i = 0; i < n_evens; ++i)
        if (pmin[i]) observe(rec, pmin[i], a + 2 * i);
    /* inject clears the bit after Phase 1 (verifier.cpp:181-183) */
    int inject_in = inject_fail >= a && inject_fail <= b && (inject_fail & 1) == 0;
    /* count_unverified + Phase 2 loop (verifier.cpp:185-200), ascending */
    for (uint64_t i = 0; i < n_evens; ++i) {
        uint64_t n = a + 2 * i;
        int verified = pmin[i] != 0 && !(inject_in && n == inject_fail);
        if (verified) continue;
        rec->unverified_p1++;
        if (n == inject_fail) {
            add_ce(rec, n);
            continue;
        }
        uint64_t p = or_phase2_resolve(n, p_small);
        if (!p) {
            add_ce(rec, n);
            continue;
        }
        rec->phase2_resolved++;
        observe(rec, p, n);
    }
    free(pmin);
    return 0;
}

static uint64_t* odd_small_primes(uint64_t p_small, uint64_t* n_out) {
    int64_t n = or_simple_sieve(p_small, NULL, 0);
    uint64_t* all = (uint64_t*)malloc((size_t)n * 8);
    or_simple_sieve(p_small, all, (uint64_t)n);
    memmove(all, all + 1, (size_t)(n - 1) * 8);
    *n_out = (uint64_t)(n - 1);
    return all;
}

int or_verify_segment(uint64_t a, uint64_t b, uint64_t cover_limit,
                      uint64_t p_small, uint64_t inject_fail,
                      gb_seg_record* rec) {
    if (p_small < 3) return -1;
    uint64_t s;
    int64_t nb = or_build_base_primes(cover_limit, NULL, 0, &s);
    if (nb < 0) return -1;
    uint32_t* base = (uint32_t*)malloc((size_t)(nb + 1) * 4);
    or_build_base_primes(cover_limit, base, (uint64_t)nb, &s);
    uint64_t n_odd;
    uint64_t* odd = odd_small_primes(p_small, &n_odd);
    int rc = or_verify_segment_tables(a, b, base, (uint64_t)nb, s, odd, n_odd,
                                      p_small, inject_fail, rec);
    free(base);
    free(odd);
    return rc;
}

/* ---- range driver: WorkPool::claim_next (pool.cpp:24-31) + merge
 *      (pool.cpp:159-174) ---- */
typedef struct {
    uint64_t start, limit, span;
    uint64_t cursor; /* atomic */
    const uint32_t* base;
    uint64_t n_base, s;
    const uint64_t* odd;
    uint64_t n_odd, p_small;
    gb_seg_record total;
    uint64_t segments;
    int error;
    pthread_mutex_t mu;
} range_ctx;

static void merge_record(gb_seg_record* t, const gb_seg_record* r) {
    t->evens_checked += r->evens_checked;
    t->unverified_p1 += r->unverified_p1;
    t->phase2_resolved += r->phase2_resolved;
    t->pmin_sum += r->pmin_sum;
    t->pmin_hash += r->pmin_hash;
    if (r->max_p != 0 &&
        (r->max_p > t->max_p || (r->max_p == t->max_p && r->max_n < t->max_n))) {
        t->max_p = r->max_p;
        t->max_n = r->max_n;
    }
    for (uint64_t i = 0; i < r->n_counterexamples && i < GB_REC_MAX_CE; ++i) {
        /* insert sorted, keep the smallest GB_REC_MAX_CE */
        uint64_t v = r->counterexamples[i];
        uint64_t n = t->n_counterexamples < GB_REC_MAX_CE ? t->n_counterexamples : GB_REC_MAX_CE;
        uint64_t k = n;
        while (k > 0 && t->counterexamples[k - 1] > v) {
            if (k < GB_REC_MAX_CE) t->counterexamples[k] = t->counterexamples[k - 1];
            --k;
        }
        if (k < GB_REC_MAX_CE) t->counterexamples[k] = v;
        t->n_counterexamples++;
    }
    if (r->n_counterexamples > GB_REC_MAX_CE)
        t->n_counterexamples += r->n_counterexamples - GB_REC_MAX_CE;
}

static void* range_worker(void* arg) {
    range_ctx* c = (range_ctx*)arg;
    for (;;) {
        uint64_t a = __atomic_fetch_add(&c->cursor, c->span, __ATOMIC_RELAXED);
        if (a < c->start || a > c->limit) break;
        uint64_t rem = c->limit - a;
        uint64_t b = a + (rem < c->span - 2 ? rem : c->span - 2);
        gb_seg_record r;
        int rc = or_verify_segment_tables(a, b, c->base, c->n_base, c->s, c->odd,
                                          c->n_odd, c->p_small, 0, &r);
        pthread_mutex_lock(&c->mu);
        if (rc) c->error = rc;
        else {
            merge_record(&c->total, &r);
            c->segments++;
        }
        pthread_mutex_unlock(&c->mu);
        if (rc) break;
    }
    return NULL;
}

int or_verify_range(uint64_t start, uint64_t limit, uint64_t seg_size,
                    uint64_t cover_limit, uint64_t p_small, int threads,
                    gb_seg_record* total, uint64_t* segments) {
    if ((start & 1) || (limit & 1) || start < 4 || start > limit) return -1;
    if (seg_size == 0 || seg_size > 0xFFFFFFFFull) return -1;
    range_ctx c;
    memset(&c, 0, sizeof(c));
    c.start = start;
    c.limit = limit;
    c.span = 2 * seg_size;
    c.cursor = start;
    c.p_small = p_small;
    int64_t nb = or_build_base_primes(cover_limit, NULL, 0, &c.s);
    uint32_t* base = (uint32_t*)malloc((size_t)(nb + 1) * 4);
    or_build_base_primes(cover_limit, base, (uint64_t)nb, &c.s);
    c.base = base;
    c.n_base = (uint64_t)nb;
    uint64_t* odd = odd_small_primes(p_small, &c.n_odd);
    c.odd = odd;
    pthread_mutex_init(&c.mu, NULL);
    if (threads < 1) threads = 1;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
    for (int i = 0; i < threads; ++i) pthread_create(&th[i], NULL, range_worker, &c);
    for (int i = 0; i < threads; ++i) pthread_join(th[i], NULL);
    free(th);
    free(base);
    free(odd);
    pthread_mutex_destroy(&c.mu);
    c.total.a = start;
    c.total.b = limit;
    *total = c.total;
    if (segments) *segments = c.segments;
    return c.error;
}
