"""Device parity against golden vectors produced by the UNMODIFIED reference
(oracle/make_goldens.py) and SURVEY.md Appendix A.  Bit-exact everywhere."""
import hashlib

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu

TOP = (1 << 64) - 1


def rec_matches(rec, want):
    got = rec.as_dict()
    for k in ("a", "b", "evens", "unverified", "phase2", "sum_pmin", "pos_hash", "max_p",
              "max_n", "n_ce", "ce"):
        assert got[k] == want[k], (k, got, want)


def test_base_primes_match_reference(gpu):
    for t in golden("base_primes.json")["tables"]:
        if t["cover"] < 1:
            continue
        with gpu.Device(t["cover"], p_small=1000) as dev:
            s, n, primes = dev.base_primes()
            assert s == t["sqrt_bound"], t["cover"]
            assert n == t["count"], t["cover"]
            if n:
                assert [int(x) for x in primes[:8]] == t["first"]
                assert [int(x) for x in primes[-8:]] == t["last"]
                assert hashlib.sha256(primes.astype("<u4").tobytes()).hexdigest() == t["sha256"]


def test_sieve_windows_match_reference(gpu):
    for w in golden("sieve_windows.json")["windows"]:
        with gpu.Device(w["cover"], p_small=1000) as dev:
            words = dev.sieve_words(w["lo"], w["hi"])
            assert int(sum(bin(int(x)).count("1") for x in words)) == w["popcount"], w
            assert hashlib.sha256(words.astype("<u8").tobytes()).hexdigest() == w["sha256"], w


def test_phase1_pmin_vectors_match_reference(gpu):
    for v in golden("pmin_vectors.json")["vectors"]:
        with gpu.Device(v["cover"], p_small=v["p_small"]) as dev:
            got = dev.phase1_pmin(v["a"], v["b"])
            want = np.array(v["pmin"], dtype=np.uint64)
            bad = np.nonzero(got != want)[0]
            assert len(bad) == 0, (v["a"], v["p_small"], bad[:5], got[bad[:5]], want[bad[:5]])


def test_small_segments_match_reference(gpu):
    for r in golden("segments_small.json")["records"]:
        with gpu.Device(r["cover"], p_small=r["p_small"], inject_fail=r["inject"]) as dev:
            rec_matches(dev.verify_segment(r["a"], r["b"]), r)


def test_c1_appendix_a(gpu):
    with gpu.Device(100_000_000) as dev:
        r = dev.verify_segment(4, 100_000_000).as_dict()
    assert r["evens"] == 49_999_999 and r["unverified"] == 0 and r["phase2"] == 0
    assert r["sum_pmin"] == 1_511_603_116
    assert r["pos_hash"] == 39_265_891_176_952_445
    assert (r["max_p"], r["max_n"]) == (1093, 60_119_912)


def test_c2_all_segments(gpu):
    recs = golden("c2_segments.json")["records"]
    with gpu.Device(10**10) as dev:
        for r in recs:
            dev.submit(r["a"], r["b"], tag=r["a"])
        for r in recs:
            got, tag = dev.wait()
            assert tag == r["a"]
            rec_matches(got, r)


def test_ceiling_window(gpu):
    r = golden("ceiling.json")["records"][0]
    with gpu.Device(r["cover"], p_small=r["p_small"], max_seg_evens=50_000) as dev:
        rec_matches(dev.verify_segment(r["a"], r["b"]), r)


def test_device_primality_matches_reference(gpu):
    vals = golden("primality.json")["values"]
    with gpu.Device(1000) as dev:
        got = dev.is_prime([v["n"] for v in vals])
    for v, g in zip(vals, got):
        assert bool(g) == v["prime"], v["n"]


def test_device_phase2_matches_reference(gpu):
    for c in golden("phase2.json")["cases"]:
        if c["p_small"] != 3 and c["n"] > 10**6:
            pass
        with gpu.Device(1000, p_small=3) as dev:
            assert dev.phase2_resolve(c["n"]) == c["p"], c


def _seg_matches(rec, r):
    got = rec.as_dict()
    for k in ("a", "b", "evens", "sum_pmin", "pos_hash", "max_p", "max_n"):
        assert got[k] == r[k], (k, got, r)
    assert got["unverified"] == 0 and got["n_ce"] == 0


def test_c3_full_range_and_anchors(gpu):
    # all of C3 through the pool (run_workers) + every 250th segment alone,
    # against the reference's Appendix A records
    g = golden("appendix_a_large.json")["c3"]
    res, _ = gpu.run_range(4, g["limit"])
    d = res.as_dict()
    for k in ("evens", "unverified", "sum_pmin", "pos_hash", "max_p", "max_n", "segments"):
        assert d[k] == g[k], (k, d, g)
    with gpu.Device(g["limit"]) as dev:
        for r in g["anchors"]:
            dev.submit(r["a"], r["b"], tag=r["a"])
        got = {}
        for _ in g["anchors"]:
            rec, tag = dev.wait()
            got[tag] = rec
    for r in g["anchors"]:
        _seg_matches(got[r["a"]], r)


def test_c5_window_first_segments(gpu):
    # base primes to 2e9 (98 M): the large-prime bitmask path, one batch of
    # 8 consecutive segments (incremental first multiples across slots)
    g = golden("appendix_a_large.json")["c5_first8"]
    with gpu.Device(g["cover"]) as dev:
        for r in g["records"]:
            dev.submit(r["a"], r["b"], tag=r["a"])
        got = {}
        for _ in g["records"]:
            rec, tag = dev.wait()
            got[tag] = rec
    tot_sum = tot_hash = 0
    for r in g["records"]:
        _seg_matches(got[r["a"]], r)
        tot_sum += got[r["a"]].as_dict()["sum_pmin"]
        tot_hash = (tot_hash + got[r["a"]].as_dict()["pos_hash"]) % (1 << 64)
    assert (tot_sum, tot_hash) == (g["sum_pmin"], g["pos_hash"])


def test_c4_sampled_segments(gpu):
    # C4 = [4, 1e13] is ~7 h of reference CPU time, so its records are
    # pinned by sampling: every 500th segment and the
    # last one, device (one batch stream at cover 1e13) vs the oracle
    import os
    from concurrent.futures import ThreadPoolExecutor

    import oracle

    limit, span = 10**13, 400_000_000
    ks = list(range(0, 25_000, 500)) + [24_999]
    segs = [(4 + k * span, min(4 + k * span + span - 2, limit)) for k in ks]
    with gpu.Device(limit) as dev:
        for a, b in segs:
            dev.submit(a, b, tag=a)
        got = {}
        for _ in segs:
            rec, tag = dev.wait()
            got[tag] = rec.as_dict()
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        want = list(ex.map(lambda ab: oracle.verify_segment(ab[0], ab[1], cover=limit).as_dict(), segs))
    for (a, b), w in zip(segs, want):
        g = got[a]
        for k in ("a", "b", "evens", "unverified", "phase2", "sum_pmin", "pos_hash", "max_p", "max_n", "n_ce"):
            assert g[k] == w[k], (k, g, w)


def test_ceiling_window_split_batch(gpu):
    # the 2^64 ceiling window as 5 pieces in ONE batch, submitted out of
    # order: base primes to 2^32 (k + p can pass 2^32 in the large-prime
    # strikes), slots above / below slot 0; the merged totals equal the
    # reference's one-segment record
    r = golden("ceiling.json")["records"][0]
    a, b = r["a"], r["b"]
    cuts = [a, a + 20_000, a + 40_002, a + 60_000, a + 80_004, b + 2]
    pieces = [(cuts[i], cuts[i + 1] - 2) for i in range(5)]
    order = [2, 0, 4, 1, 3]
    with gpu.Device(r["cover"], p_small=r["p_small"]) as dev:
        for i in order:
            dev.submit(*pieces[i], tag=i)
        recs = [None] * 5
        for _ in order:
            rec, tag = dev.wait()
            recs[tag] = rec.as_dict()
    M = 1 << 64
    assert sum(x["evens"] for x in recs) == r["evens"]
    assert sum(x["unverified"] for x in recs) == 0 and sum(x["n_ce"] for x in recs) == 0
    assert sum(x["sum_pmin"] for x in recs) % M == r["sum_pmin"]
    assert sum(x["pos_hash"] for x in recs) % M == r["pos_hash"]
    best = max(recs, key=lambda x: (x["max_p"], -x["max_n"]))
    assert (best["max_p"], best["max_n"]) == (r["max_p"], r["max_n"])
