"""Time one verification pass over evens [start, start + span] (default: a
C5-style window near 4e18) through the pool, device resident; prints the
merged record and the per-kernel device times.

    python tools/range_bench.py [start] [span] [reps]
"""
import sys
import time

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2603_07850_b200 as gb

start = int(float(sys.argv[1])) if len(sys.argv) > 1 else 4 * 10**18
span = int(float(sys.argv[2])) if len(sys.argv) > 2 else 10**10
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
start += start & 1
limit = start + span
t0 = time.time()
dev = gb.Device(limit)
print(f"open {time.time() - t0:.3f}s", flush=True)
dev.set_timing(True)
for rep in range(reps):
    pool = gb.Pool(start, limit, 200_000_000)
    t = time.perf_counter()
    r = gb.drain_pool(dev, pool)
    dt = time.perf_counter() - t
    d = r.as_dict()
    print(f"[{start}, {limit}] time={dt:.3f}s rate={d['evens'] / dt:.4e}/s {d}", flush=True)
print("kernel ms/launches [verify, ?, large-strike/offsets, stragglers]:", dev.kernel_times(reset=True))
