"""Times the pieces of bench.py's e2e step (open / drain / close)."""
import sys, time
sys.path.insert(0, '/root/repo')
import paper_2603_07850_b200 as gb
limit = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**12
for rep in range(4):
    t0 = time.perf_counter()
    dev = gb.Device(limit)
    t1 = time.perf_counter()
    pool = gb.Pool(4, limit, 200_000_000)
    r = gb.drain_pool(dev, pool)
    t2 = time.perf_counter()
    dev.close()
    t3 = time.perf_counter()
    print(f"open {t1-t0:.3f} drain {t2-t1:.3f} close {t3-t2:.3f} evens {r.evens_checked}", flush=True)
dev = gb.Device(limit)
for rep in range(3):
    pool = gb.Pool(4, limit, 200_000_000)
    t1 = time.perf_counter(); r = gb.drain_pool(dev, pool); t2 = time.perf_counter()
    print(f"resident drain {t2-t1:.3f}")
