#!/usr/bin/env python3
"""Generate tests/golden/*.json from the UNMODIFIED reference.

The reference library is compiled in place by oracle/build_ref.sh into
oracle/_ref/libref.so; every vector below comes from the reference's own
functions (verify_segment, phase1_verify(..., min_primes_out),
tiled_sieve_segment, build_base_primes, phase2_resolve, is_prime_u64).
TEST INFRASTRUCTURE ONLY.  Needs /root/reference (this container), so the
fixtures are committed; the GPU box only reads them.

usage: python oracle/make_goldens.py [--quick]
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import random
import sys
import time
from concurrent.futures import ProcessPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")
TOP = (1 << 64) - 1


def words_digest(words) -> str:
    return hashlib.sha256(words.astype("<u8").tobytes()).hexdigest()


def seg_job(args):
    a, b, cover, p_small, inject = args
    r = O.ref_segment_record(a, b, cover, p_small, inject)
    d = r.as_dict()
    d.update(cover=cover, p_small=p_small, inject=inject)
    return d


def pmin_job(args):
    a, b, cover, p_small = args
    v = O.ref_phase1_pmin(a, b, p_small, cover)
    return dict(a=a, b=b, cover=cover, p_small=p_small, pmin=[int(x) for x in v])


def sieve_job(args):
    lo, hi, cover, tile = args
    w = O.ref_sieve_words(lo, hi, cover, tile)
    pop = int(sum(bin(int(x)).count("1") for x in w))
    return dict(lo=lo, hi=hi, cover=cover, tile=tile, popcount=pop, sha256=words_digest(w))


def base_job(cover):
    import ctypes as C
    import numpy as np
    s = C.c_uint64()
    n = O.ref().ref_base_primes(cover, None, 0, C.byref(s))
    out = np.zeros(max(n, 1), dtype=np.uint32)
    O.ref().ref_base_primes(cover, out.ctypes.data_as(C.POINTER(C.c_uint32)), n, C.byref(s))
    out = out[:n]
    return dict(cover=cover, sqrt_bound=int(s.value), count=int(n),
                first=[int(x) for x in out[:8]], last=[int(x) for x in out[-8:]],
                sha256=hashlib.sha256(out.astype("<u4").tobytes()).hexdigest())


def dump(name, obj):
    os.makedirs(GOLD, exist_ok=True)
    path = os.path.join(GOLD, name)
    with open(path, "w") as f:
        json.dump(obj, f, indent=1)
    print(f"wrote {path}", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true", help="skip the slow C2 / ceiling sets")
    ap.add_argument("--jobs", type=int, default=os.cpu_count())
    args = ap.parse_args()
    if not O.ref_available():
        sys.exit("oracle/_ref/libref.so missing: run oracle/build_ref.sh first")
    ex = ProcessPoolExecutor(args.jobs)
    prov = {"generator": "oracle/make_goldens.py",
            "source": "UNMODIFIED reference /root/reference/proj compiled by oracle/build_ref.sh",
            "generated": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}

    # ---- small segments: known-answer cases of the reference tests + random
    rng = random.Random(0xacce972)  # acceptance.cpp:89 seed
    jobs = [
        (4, 20, 1000, 1000, 0),                 # test_verifier.cpp:59-73
        (4, 4, 100, 3, 0),                      # :75-84
        (4, 10_000, 1_000_000, 1_000_000, 0),   # :265-282 (173 @ 7426)
        (4, 20_000, 20_000, 3, 0),              # :284-304 phase 2 routing
        (4, 10_000, 10_000, 1000, 5000),        # :306-323 inject
        (4, 100_000, 100_000, 1_000_000, 4148), # test_cli.cpp:176-195 inject 4148
        (4, 1_000_000, 1_000_000, 1_000_000, 0),  # acceptance c4 range
        (1_000_000_000_000, 1_000_000_000_400, 1_000_000_000_402, 1_000_000, 0),  # :330-349
        (4, 200, 200, 3, 0), (6, 6, 6, 3, 0), (8, 8, 8, 3, 8), (4, 64, 64, 5, 0),
        (1_000_002, 1_200_000, 1_200_000, 1_000_000, 0),  # SPEC boundary coverage case
    ]
    for _ in range(40):  # random small segments, random p_small, some injects
        a = 4 + 2 * rng.randrange(0, 5_000_000)
        b = a + 2 * rng.randrange(0, 30_000)
        p_small = rng.choice([3, 5, 7, 11, 97, 128, 129, 131, 1000, 8191, 8193, 1_000_000])
        inject = 0 if rng.random() < 0.7 else a + 2 * rng.randrange(0, (b - a) // 2 + 1)
        cover = b + 2 * rng.randrange(0, 1000)
        jobs.append((a, b, cover, p_small, inject))
    for base in (10**10, 10**12, 10**13, 10**15, 4 * 10**18, 10**19):
        for k in range(3):
            a = base + 2 * rng.randrange(0, 10**6) + 2 * 10**6 * k
            b = a + 2 * rng.randrange(10_000, 40_000)
            jobs.append((a, b, b, 1_000_000, 0))
    segs = list(ex.map(seg_job, jobs))
    dump("segments_small.json", {"provenance": prov, "records": segs})

    # ---- per-n Phase 1 minimal primes (phase1_verify min_primes_out)
    pj = [(4, 20, 1000, 1000), (4, 2000, 2000, 2000), (4, 20_000, 20_000, 3),
          (4, 20_000, 20_000, 131), (10**12, 10**12 + 400, 10**12 + 402, 1_000_000),
          (10**12, 10**12 + 40_000, 10**12 + 40_000, 1_000_000),
          (10**13, 10**13 + 40_000, 10**13 + 40_000, 1_000_000),
          (4 * 10**18, 4 * 10**18 + 20_000, 4 * 10**18 + 20_000, 1_000_000),
          (123_456_789_012, 123_456_789_012 + 30_000, 123_456_789_012 + 30_000, 1_000_000)]
    pm = list(ex.map(pmin_job, pj))
    dump("pmin_vectors.json", {"provenance": prov, "vectors": pm})

    # ---- sieve windows (tiled_sieve_segment words)
    sj = [(3, 31, 31, 32768), (1, 9, 9, 32768), (3, 99, 99, 32768),
          (1_000_001, 2_999_999, 3_000_000, 64), (1_000_001, 2_999_999, 3_000_000, 32768),
          (10**12 + 1, 10**12 + 20_001, 10**12 + 20_001, 32768),
          (10**13 + 1, 10**13 + 2_000_001, 10**13 + 2_000_001, 32768),
          (4 * 10**18 + 1, 4 * 10**18 + 400_001, 4 * 10**18 + 400_001, 32768)]
    rng2 = random.Random(0x5e95eed)  # test_sieve.cpp:152 seed
    for _ in range(30):
        lo = rng2.randrange(0, 9_000_000) + 1
        lo |= 1
        hi = lo + 2 * rng2.randrange(0, 50_000)
        sj.append((lo, hi, 10_000_000, 32768))
    sv = list(ex.map(sieve_job, sj))
    dump("sieve_windows.json", {"provenance": prov, "windows": sv})

    # ---- base primes (build_base_primes)
    covers = [1, 4, 11, 12, 31, 99, 1000, 10**8, 10**10, 10**12, 10**13,
              4 * 10**18 + 10**11]
    bp = list(ex.map(base_job, covers))
    dump("base_primes.json", {"provenance": prov, "tables": bp})

    # ---- primality fixed points (is_prime_u64)
    vals = [0, 1, 2, 3, 4, 561, 25326001, (1 << 61) - 1, TOP, 18446744073709551557,
            3215031751, 2152302898747, 3474749660383, 341550071728321,
            3825123056546413051, 318665857834031151167461 % (1 << 64)]
    r3 = random.Random(0x5eed03)
    vals += [r3.getrandbits(64) for _ in range(2000)]
    vals += list(range(TOP - 2000, TOP + 1))
    pr = [dict(n=v, prime=bool(O.ref().ref_is_prime(v))) for v in vals]
    dump("primality.json", {"provenance": prov, "values": pr})

    # ---- Phase 2 resolver (phase2_resolve, table disabled)
    p2 = []
    for n, ps in [(4, 3), (6, 3), (8, 3), (100, 3), (100, 1000), (TOP - 1, 1_000_000),
                  (1_000_000_000_008, 1000), (98, 3), (128, 3), (1_000_000, 3)]:
        import ctypes as C
        p = C.c_uint64()
        O.ref().ref_phase2_resolve(n, ps, C.byref(p))
        p2.append(dict(n=n, p_small=ps, p=int(p.value)))
    dump("phase2.json", {"provenance": prov, "cases": p2})

    if not args.quick:
        # C2: all 25 segments of [4, 1e10] with the default segmentation
        span = 400_000_000
        c2 = []
        a = 4
        while a <= 10**10:
            b = a + min(10**10 - a, span - 2)
            c2.append((a, b, 10**10, 1_000_000, 0))
            a += span
        recs = list(ex.map(seg_job, c2))
        dump("c2_segments.json", {"provenance": prov, "limit": 10**10, "records": recs})
        # acceptance c7: the ceiling window, one 50,000-even segment
        cj = [(TOP - 99_999, TOP - 1, TOP - 1, 1_000_000, 0)]
        dump("ceiling.json", {"provenance": prov, "records": list(ex.map(seg_job, cj))})
    ex.shutdown()


if __name__ == "__main__":
    main()
