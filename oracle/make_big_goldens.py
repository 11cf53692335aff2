#!/usr/bin/env python3
"""Per-segment reference records for the north-star configurations C4 and C5.

C4 = every segment of [4, 1e13]               (25,000 segments, cover 1e13)
C5 = every segment of [4e18, 4e18 + 1e11]     (251 segments, cover 4e18+1e11)

Every record comes from the UNMODIFIED reference library
(oracle/_ref/libref.so, built by oracle/build_ref.sh) through
ref_segment_record1: sieve_range_for -> tiled_sieve_segment -> phase1_verify
(min_primes_out) -> count_unverified -> phase2_resolve, the composition of
verify_segment (verifier.cpp:167-206).  Segmentation follows
WorkPool::claim_next (pool.cpp:24-31) with seg_size 2e8, p_small 1e6.

The run is long (C4 is ~55 core-hours), so it is resumable: records are
appended to oracle/_big/<set>.tsv as they complete and the committed
fixture tests/golden/<set>_segments.tsv.gz is (re)written from it by
`--pack`.  Segments are processed in a stride order (every 10th segment
first, then every 5th, ...) so a partial file is still an even sample of
the whole range.  TEST INFRASTRUCTURE ONLY.

usage:
  python oracle/make_big_goldens.py --set c5 --jobs 7
  python oracle/make_big_goldens.py --set c4 --jobs 7
  python oracle/make_big_goldens.py --pack
  python oracle/make_big_goldens.py --selfcheck   # record1 == verify_segment record
"""
from __future__ import annotations

import argparse
import gzip
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor, as_completed

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

BIG = os.path.join(HERE, "_big")
GOLD = os.path.join(ROOT, "tests", "golden")
SEG = 200_000_000
P_SMALL = 1_000_000

SETS = {
    "c4": dict(start=4, limit=10**13, cover=10**13),
    "c5": dict(start=4 * 10**18, limit=4 * 10**18 + 10**11, cover=4 * 10**18 + 10**11),
}
COLS = ["idx", "a", "b", "evens", "unverified", "phase2", "sum_pmin", "pos_hash",
        "max_p", "max_n", "n_ce"]


def segments(start: int, limit: int):
    """WorkPool::claim_next (pool.cpp:24-31) with the subtraction forms."""
    span = 2 * SEG
    out = []
    a = start
    idx = 0
    while a <= limit:
        b = a + min(limit - a, span - 2)
        out.append((idx, a, b))
        idx += 1
        if limit - a < span:
            break
        a += span
    return out


def stride_order(n: int):
    seen = set()
    order = []
    for stride in (10, 5, 2, 1):
        for i in range(0, n, stride):
            if i not in seen:
                seen.add(i)
                order.append(i)
    if n - 1 not in seen:
        order.append(n - 1)
    return order


def job(args):
    idx, a, b, cover = args
    t0 = time.time()
    r = O.ref_segment_record1(a, b, cover, P_SMALL, 0)
    return (idx, a, b, r.evens_checked, r.unverified_p1, r.phase2_resolved, r.pmin_sum,
            r.pmin_hash, r.max_p, r.max_n, r.n_counterexamples), time.time() - t0


def load(path: str):
    done = {}
    if os.path.exists(path):
        with open(path) as f:
            for line in f:
                if line.startswith("#") or not line.strip():
                    continue
                v = [int(x) for x in line.split()]
                if len(v) == len(COLS):
                    done[v[0]] = tuple(v)
    return done


def run_set(name: str, jobs: int, stride: int = 1, part=None, out=None, skip=None):
    cfg = SETS[name]
    segs = segments(cfg["start"], cfg["limit"])
    os.makedirs(BIG, exist_ok=True)
    path = out or os.path.join(BIG, f"{name}.tsv")
    done = load(path)
    if skip:  # records already produced elsewhere (e.g. on another host)
        for p in skip:
            done.update(load(p))
    lo, hi = part if part else (0, len(segs))
    todo = [segs[i] for i in stride_order(len(segs))
            if lo <= i < hi and segs[i][0] not in done and (i % stride == 0 or i == len(segs) - 1)]
    print(f"{name}: {len(segs)} segments, {len(done)} done, {len(todo)} to go", flush=True)
    t0 = time.time()
    with ProcessPoolExecutor(jobs) as ex, open(path, "a") as f:
        # submit in windows so the stride order is respected on completion
        pending = set()
        it = iter(todo)
        n = 0
        def fill():
            for _ in range(2 * jobs - len(pending)):
                s = next(it, None)
                if s is None:
                    return
                pending.add(ex.submit(job, (s[0], s[1], s[2], cfg["cover"])))
        fill()
        while pending:
            for fut in as_completed(list(pending)):
                pending.remove(fut)
                row, dt = fut.result()
                f.write(" ".join(str(x) for x in row) + "\n")
                f.flush()
                n += 1
                if n % 50 == 0:
                    el = time.time() - t0
                    print(f"{name}: {n}/{len(todo)} in {el:.0f}s (last seg {dt:.1f}s)", flush=True)
                fill()
                break


def pack():
    for name, cfg in SETS.items():
        path = os.path.join(BIG, f"{name}.tsv")
        done = load(path)
        if not done:
            continue
        total = len(segments(cfg["start"], cfg["limit"]))
        out = os.path.join(GOLD, f"{name}_segments.tsv.gz")
        with gzip.GzipFile(out, "wb", mtime=0) as g:
            hdr = (f"# {name}: reference per-segment records (oracle/make_big_goldens.py; "
                   f"UNMODIFIED reference via oracle/_ref/libref.so ref_segment_record1)\n"
                   f"# start={cfg['start']} limit={cfg['limit']} cover={cfg['cover']} "
                   f"seg_size={SEG} p_small={P_SMALL} segments_total={total} "
                   f"segments_here={len(done)}\n# " + " ".join(COLS) + "\n")
            g.write(hdr.encode())
            for idx in sorted(done):
                g.write((" ".join(str(x) for x in done[idx]) + "\n").encode())
        print(f"wrote {out}: {len(done)}/{total}")


def selfcheck():
    """ref_segment_record1 must equal the verify_segment-based record."""
    cases = [(4, 10_000, 10**6, 10**6, 0), (4, 20_000, 20_000, 3, 0),
             (4, 10_000, 10_000, 1000, 5000), (4, 100_000, 100_000, 10**6, 4148),
             (10**12, 10**12 + 400_000, 10**12 + 400_000, 10**6, 0),
             (4 * 10**18, 4 * 10**18 + 200_000, 4 * 10**18 + 200_000, 10**6, 0)]
    for a, b, cover, ps, inj in cases:
        r0 = O.ref_segment_record(a, b, cover, ps, inj).key()
        r1 = O.ref_segment_record1(a, b, cover, ps, inj).key()
        assert r0 == r1, (a, b, r0, r1)
    print("selfcheck ok")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--set", choices=sorted(SETS))
    ap.add_argument("--jobs", type=int, default=max(1, (os.cpu_count() or 2) - 1))
    ap.add_argument("--stride", type=int, default=1, help="only every k-th segment (+ the last)")
    ap.add_argument("--part", help="only segment indices i0:i1")
    ap.add_argument("--out", help="records file (default oracle/_big/<set>.tsv)")
    ap.add_argument("--skip", action="append", help="records files whose segments are done")
    ap.add_argument("--merge", action="append", help="records files to merge into oracle/_big/<set>.tsv")
    ap.add_argument("--pack", action="store_true")
    ap.add_argument("--selfcheck", action="store_true")
    a = ap.parse_args()
    if not O.ref_available():
        sys.exit("oracle/_ref/libref.so missing: run oracle/build_ref.sh first")
    if a.selfcheck:
        selfcheck()
    if a.set and a.merge:
        path = os.path.join(BIG, f"{a.set}.tsv")
        done = load(path)
        n0 = len(done)
        for p in a.merge:
            done.update(load(p))
        with open(path, "w") as f:
            for idx in sorted(done):
                f.write(" ".join(str(x) for x in done[idx]) + "\n")
        print(f"merged: {n0} -> {len(done)} records")
    elif a.set:
        part = tuple(int(x) for x in a.part.split(":")) if a.part else None
        run_set(a.set, a.jobs, a.stride, part, a.out, a.skip)
    if a.pack:
        pack()


if __name__ == "__main__":
    main()
