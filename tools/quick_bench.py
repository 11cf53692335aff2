import sys, time
sys.path.insert(0, '/root/repo')
import paper_2603_07850_b200 as gb
limit = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**12
t0 = time.time()
dev = gb.Device(limit)
t1 = time.time()
print("open", t1 - t0, "bucket", dev.bucket_info(), flush=True)
span = 400_000_000
depth = dev.max_inflight()
dev.set_timing(True)
def run():
    a = 4; inflight = 0; tot = None; segs = 0
    evens = 0; sp = 0; sh = 0; mx = (0, 0)
    t = time.time()
    while a <= limit or inflight:
        while a <= limit and inflight < depth:
            b = a + min(limit - a, span - 2)
            dev.submit(a, b, a); a += span; inflight += 1
        r, _ = dev.wait(); inflight -= 1; segs += 1
        evens += r.evens_checked; sp = (sp + r.pmin_sum) % 2**64; sh = (sh + r.pmin_hash) % 2**64
        if r.max_p > mx[0] or (r.max_p == mx[0] and r.max_n < mx[1]): mx = (r.max_p, r.max_n)
    return time.time() - t, segs, evens, sp, sh, mx
for rep in range(2):
    dt, segs, evens, sp, sh, mx = run()
    print(f"limit={limit:.0e} time={dt:.3f}s segs={segs} evens={evens} rate={evens/dt:.4e}/s sum={sp} hash={sh} max={mx}", flush=True)
print("kernel times", dev.kernel_times(reset=True), "launches", dev.launch_count())
try:
    import ctypes as C
    v = (C.c_uint64 * 8)()
    if gb.lib().gb_debug_stats(v, 1) == 0:
        print("stats [generic evens, inplace deep, queued deep, deep rounds, stragglers, fast blocks, generic blocks]:", list(v))
except Exception as e:
    print("no stats:", e)
