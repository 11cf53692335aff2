"""CPU: pin the oracle (oracle/oracle.c, the C restatement of the reference
path) against golden vectors produced by the UNMODIFIED reference
(oracle/make_goldens.py -> tests/golden/*.json) and the reference's own
known-answer tests.  No GPU."""
import hashlib
import os

import numpy as np
import pytest

import oracle
from conftest import GOLD, golden


def test_known_answers_from_reference_tests():
    # pi(1e6) = 78,498 (test_sieve.cpp:29-31); 24 odd primes in [3,99]
    # (test_sieve.cpp:139-147)
    small = oracle.simple_sieve(1_000_000)
    assert len(small) == 78_498 and small[0] == 2 and small[-1] == 999_983
    w = oracle.sieve_words(3, 99, cover=99)
    assert sum(bin(int(x)).count("1") for x in w) == 24
    # tile-size independence: popcount 138,318 on [1,000,001, 2,999,999]
    # (test_sieve.cpp:163-177)
    for tile in (64, 4096, 32768, 1 << 20):
        w = oracle.sieve_words(1_000_001, 2_999_999, odds_per_tile=tile)
        assert sum(bin(int(x)).count("1") for x in w) == 138_318
    # sieve_range_for fixed points (test_verifier.cpp:23-37)
    assert oracle.sieve_range_for(4, 20, 1000) == (3, 17)
    # primality fixed points (test_primality.cpp:59-70)
    for n, p in [(561, False), (25326001, False), ((1 << 61) - 1, True),
                 (18446744073709551557, True), (2, True), (1, False), (0, False)]:
        assert oracle.is_prime(n) == p, n


def test_pmin_small_fixed_points():
    # p_min on [4,20] = {2,3,3,3,5,3,3,5,3} (test_verifier.cpp:59-73)
    got = oracle.phase1_pmin(4, 20, p_small=1000, cover=1000)
    assert [int(x) for x in got] == [2, 3, 3, 3, 5, 3, 3, 5, 3]
    # [4, 1e4]: max 173 @ 7426, 4,999 evens (test_verifier.cpp:265-282)
    r = oracle.verify_segment(4, 10_000, cover=10_000).as_dict()
    assert (r["evens"], r["max_p"], r["max_n"]) == (4_999, 173, 7426)
    # Phase 2 at 2^64-2 gives p = 277 (test_verifier.cpp:209-219)
    assert oracle.phase2_resolve((1 << 64) - 2, 1_000_000) == 277


def test_base_primes_golden():
    for t in golden("base_primes.json")["tables"]:
        if t["cover"] < 1 or t["count"] > 5_000_000:
            continue
        s, primes = oracle.base_primes(t["cover"])
        assert s == t["sqrt_bound"] and len(primes) == t["count"], t["cover"]
        if len(primes):
            assert hashlib.sha256(primes.astype("<u4").tobytes()).hexdigest() == t["sha256"]


def test_sieve_windows_golden():
    for w in golden("sieve_windows.json")["windows"]:
        if (w["hi"] - w["lo"]) > 50_000_000 or w["cover"] > 10**13:
            continue
        words = oracle.sieve_words(w["lo"], w["hi"], cover=w["cover"])
        assert hashlib.sha256(words.astype("<u8").tobytes()).hexdigest() == w["sha256"], w


def test_pmin_vectors_golden():
    for v in golden("pmin_vectors.json")["vectors"]:
        if v["a"] > 10**14:
            continue  # base primes to 2e9: covered on the GPU side
        got = oracle.phase1_pmin(v["a"], v["b"], p_small=v["p_small"], cover=v["cover"])
        assert np.array_equal(got, np.array(v["pmin"], dtype=np.uint64)), v["a"]


def test_segments_small_golden():
    for r in golden("segments_small.json")["records"]:
        if r["cover"] > 10**13:
            continue
        got = oracle.verify_segment(r["a"], r["b"], cover=r["cover"], p_small=r["p_small"],
                                    inject_fail=r["inject"]).as_dict()
        for k in ("evens", "unverified", "phase2", "sum_pmin", "pos_hash", "max_p", "max_n",
                  "n_ce", "ce"):
            assert got[k] == r[k], (k, got, r)


def test_primality_golden():
    for v in golden("primality.json")["values"]:
        assert oracle.is_prime(v["n"]) == v["prime"], v["n"]


def test_phase2_golden():
    for c in golden("phase2.json")["cases"]:
        assert oracle.phase2_resolve(c["n"], c["p_small"]) == c["p"], c


def test_c1_appendix_a():
    """C1 [4, 1e8] = one segment."""
    r = oracle.verify_segment(4, 100_000_000, cover=100_000_000).as_dict()
    assert r["evens"] == 49_999_999 and r["unverified"] == 0
    assert r["sum_pmin"] == 1_511_603_116 and r["pos_hash"] == 39_265_891_176_952_445
    assert (r["max_p"], r["max_n"]) == (1093, 60_119_912)


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_oracle_matches_compiled_reference_random_segments():
    """The restatement against the compiled reference on random small
    segments (seed 0xacce972 as acceptance.cpp:89)."""
    rng = np.random.default_rng(0xACCE972)
    for _ in range(40):
        a = int(rng.integers(2, 5_000_000)) * 2
        b = a + 2 * int(rng.integers(0, 20_000))
        want = oracle.ref_segment_record(a, b, b, 1_000_000, 0)
        got = oracle.verify_segment(a, b, cover=b)
        assert got.key() == want.key(), (a, b)


def _big(name):
    import gzip
    path = os.path.join(GOLD, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not generated")
    meta, rows = {}, []
    with gzip.open(path, "rt") as f:
        for line in f:
            if line.startswith("#"):
                meta.update(dict(t.split("=", 1) for t in line[1:].split() if "=" in t))
                continue
            if line.strip():
                rows.append([int(x) for x in line.split()])
    return {k: int(v) for k, v in meta.items()}, rows


@pytest.mark.parametrize("name", ["c4_segments.tsv.gz", "c5_segments.tsv.gz"])
def test_big_golden_files_follow_claim_rule(name):
    """The C4/C5 reference records are WorkPool claims (pool.cpp:24-31):
    segment idx is [start + idx * 2 seg, min(that + 2 seg - 2, limit)]."""
    meta, rows = _big(name)
    span = 2 * meta["seg_size"]
    for r in rows:
        a = meta["start"] + r[0] * span
        assert (r[1], r[2]) == (a, min(a + span - 2, meta["limit"]))
        assert r[3] == (r[2] - r[1]) // 2 + 1 and r[4] == 0 and r[10] == 0


def test_oracle_matches_a_c4_reference_record():
    """The C restatement against one reference record at the top of C4
    (cover 1e13): the oracle is pinned at the north-star height too."""
    meta, rows = _big("c4_segments.tsv.gz")
    r = max(rows, key=lambda v: v[0])
    got = oracle.verify_segment(r[1], r[2], cover=meta["cover"], p_small=meta["p_small"])
    assert got.key()[:10] == tuple(r[1:])
