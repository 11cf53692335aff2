"""The north-star configurations against the UNMODIFIED reference, record by
record: C4 = every segment of [4, 1e13] and C5 = every segment of
[4e18, 4e18 + 1e11] (tests/golden/c4_segments.tsv.gz, c5_segments.tsv.gz,
written by oracle/make_big_goldens.py from oracle/_ref/libref.so, i.e.
verify_segment's composition verifier.cpp:167-206 per WorkPool claim
pool.cpp:24-31).  Every record the golden file holds is compared bit-exactly
(evens, unverified, Phase 2 count, checksum, hash, MinPrimeMax,
counterexamples); when the file holds every segment the merged totals
(pool.cpp:159-174) are compared too."""
import gzip
import os

import pytest

from conftest import GOLD

pytestmark = pytest.mark.gpu

M = (1 << 64) - 1


def load(name):
    path = os.path.join(GOLD, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not generated")
    meta, rows = {}, []
    with gzip.open(path, "rt") as f:
        for line in f:
            if line.startswith("#"):
                for tok in line[1:].split():
                    if "=" in tok:
                        k, v = tok.split("=", 1)
                        meta[k] = int(v)
                continue
            v = [int(x) for x in line.split()]
            if v:
                rows.append(v)
    return meta, rows


def run_all(gpu, meta, rows):
    """Every golden segment through the asynchronous boundary, pipelined."""
    want = {r[0]: r for r in rows}
    got = {}
    with gpu.Device(meta["cover"], p_small=meta["p_small"], max_seg_evens=meta["seg_size"]) as dev:
        depth = dev.max_inflight()
        pend = 0
        for r in rows:
            dev.submit(r[1], r[2], r[0])
            pend += 1
            if pend >= depth:
                rec, tag = dev.wait()
                got[tag] = rec
                pend -= 1
        while pend:
            rec, tag = dev.wait()
            got[tag] = rec
            pend -= 1
    bad = []
    for idx, r in want.items():
        d = got[idx].as_dict()
        g = (d["a"], d["b"], d["evens"], d["unverified"], d["phase2"], d["sum_pmin"], d["pos_hash"],
             d["max_p"], d["max_n"], d["n_ce"])
        if g != tuple(r[1:]):
            bad.append((idx, g, r))
    assert not bad, f"{len(bad)} of {len(want)} records differ, first: {bad[:3]}"
    return got


def totals(rows):
    t = dict(evens=0, unverified=0, phase2=0, sum=0, hash=0, max_p=0, max_n=0, n_ce=0)
    for r in rows:
        t["evens"] += r[3]
        t["unverified"] += r[4]
        t["phase2"] += r[5]
        t["sum"] = (t["sum"] + r[6]) & M
        t["hash"] = (t["hash"] + r[7]) & M
        if r[8] > t["max_p"] or (r[8] == t["max_p"] and r[8] and r[9] < t["max_n"]):
            t["max_p"], t["max_n"] = r[8], r[9]
        t["n_ce"] += r[10]
    return t


@pytest.mark.parametrize("name,n_total,evens", [
    ("c5_segments.tsv.gz", 251, 50_000_000_001),
    ("c4_segments.tsv.gz", 25_000, 4_999_999_999_999),
])
def test_north_star_range_records(gpu, name, n_total, evens):
    meta, rows = load(name)
    assert meta["segments_total"] == n_total
    assert len(rows) == meta["segments_here"] and len(rows) > 0
    run_all(gpu, meta, rows)
    if len(rows) == n_total:
        t = totals(rows)
        assert t["evens"] == evens and t["unverified"] == 0 and t["n_ce"] == 0
        # the whole range through the pool on the device: the same totals
        import paper_2603_07850_b200 as gb
        with gb.Device(meta["limit"], p_small=meta["p_small"], max_seg_evens=meta["seg_size"]) as dev:
            pool = gb.Pool(meta["start"], meta["limit"], meta["seg_size"])
            r = gb.drain_pool(dev, pool).as_dict()
        assert (r["evens"], r["sum_pmin"], r["pos_hash"], r["max_p"], r["max_n"], r["segments"]) == \
            (t["evens"], t["sum"], t["hash"], t["max_p"], t["max_n"], n_total)
