/*
 * goldbach_b200_pool.h -- C-ABI of the work-stealing pool and the range
 * runner (the layer above verify_segment).
 *
 * Reference interfaces replaced:
 *   WorkPool ctor / claim_next         proj/include/goldbach/pool.hpp:21-42,
 *                                      proj/src/pool.cpp:13-31
 *   run_workers worker loop + merge    proj/src/pool.cpp:70-175
 *   RunResult                          proj/include/goldbach/pool.hpp:114-123
 *
 * B200 changes: a worker is one GPU (gb_dev); the pool cursor may live in
 * POSIX shared memory so that several processes on one node (one per GPU,
 * torchrun) steal segments from ONE atomic counter, exactly the claim
 * semantics of pool.cpp:24-31.  Per-GPU results are merged with the
 * reference's rules (sums, MinPrimeMax, sorted counterexamples).
 */
#ifndef GOLDBACH_B200_POOL_H
#define GOLDBACH_B200_POOL_H

#include <stdint.h>

#include "goldbach_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gb_pool gb_pool;

/* RunResult (pool.hpp:114-123) plus the checksum and the segment count. */
typedef struct gb_run_result {
    uint64_t evens_checked;
    uint64_t unverified_total;
    uint64_t phase2_total;
    uint64_t pmin_sum;
    uint64_t pmin_hash;
    uint64_t max_p, max_n;       /* MinPrimeMax */
    uint64_t segments;
    uint64_t n_counterexamples;  /* exact; the smallest GB_REC_MAX_CE kept */
    uint64_t counterexamples[GB_REC_MAX_CE];
    double wall_seconds;
} gb_run_result;

/* WorkPool(start, limit, seg_size) (pool.cpp:13-22): start/limit even,
 * 4 <= start <= limit, 1 <= seg_size <= 2^32-1 (else GB_ERR_PARAM).
 * shm_name == NULL: process-local cursor.  Otherwise the cursor lives in the
 * POSIX shared-memory object `shm_name`; create=1 creates/initialises it
 * (one process), create=0 attaches to an existing one. */
int gb_pool_create(uint64_t start, uint64_t limit, uint64_t seg_size,
                   const char* shm_name, int create, gb_pool** out);

/* claim_next (pool.cpp:24-31): 1 and the job, 0 when exhausted, <0 = -status. */
int gb_pool_claim(gb_pool* pool, uint64_t* a, uint64_t* b, uint64_t* index);

/* Cooperative stop (pool.cpp:104-111): after gb_pool_request_stop every
 * claim on this pool -- in every process attached to a shared cursor --
 * returns 0.  Workers set it when a segment has counterexamples.
 * gb_pool_stop_requested returns 1 once set. */
int gb_pool_request_stop(gb_pool* pool);
int gb_pool_stop_requested(const gb_pool* pool);

/* Frees the handle; unlink=1 also removes the shared-memory object. */
int gb_pool_destroy(gb_pool* pool, int unlink);

/* One GPU worker (pool.cpp:90-120) on an open device: claims segments until
 * the pool is exhausted or stopped (a counterexample here sets the pool's
 * stop, which every attached rank honours), keeps up to
 * max_inflight segments in flight (0 = device maximum; slow start from 1),
 * and returns this worker's merged result. */
int gb_drain_pool(gb_dev* dev, gb_pool* pool, int max_inflight, gb_run_result* out);

/* run_workers (pool.cpp:70-175) in-process: n_workers GPU workers mapped
 * round-robin onto devices[0..n_devices), one host thread each, tables
 * built for cover_limit = limit (cli.cpp:314).  per_worker_segments (may be
 * NULL) receives n_workers counts. */
int gb_run_range(uint64_t start, uint64_t limit, uint64_t seg_size, uint64_t p_small,
                 uint64_t inject_fail, const int* devices, int n_devices, int n_workers,
                 int progress, gb_run_result* out, uint64_t* per_worker_segments);

/* Device bytes one worker handle allocates for (cover_limit, p_small,
 * max_seg_evens): the per-GPU term of validate_resources (cli.cpp:264-296). */
uint64_t gb_estimate_device_bytes(uint64_t cover_limit, uint64_t p_small,
                                  uint64_t max_seg_evens);

/* Message of the last failing pool / run call on this thread. */
const char* gb_pool_last_error(void);

/* Creates device's primary CUDA context (cudaSetDevice + cudaFree(0)).  The
 * CLI calls it for every worker GPU on background threads while it checks
 * resources, so context creation overlaps the check.  Not part of the
 * reference interface. */
int gb_warm_device(int device);

/* Free / total memory of a device: NVML (no CUDA context needed), else
 * cudaMemGetInfo. */
int gb_device_memory(int device, uint64_t* free_bytes, uint64_t* total_bytes);

#ifdef __cplusplus
}
#endif

#endif /* GOLDBACH_B200_POOL_H */
