import sys, time
sys.path.insert(0, '.')
import paper_2603_07850_b200 as gb
from paper_2603_07850_b200 import dist as gd
limit = 10**12
dev = gb.Device(limit)
pool = gb.Pool(4, limit, 200_000_000); gb.drain_pool(dev, pool); pool.close(unlink=False)
for k in range(3):
    t0 = time.perf_counter()
    pool = gb.Pool(4, limit, 200_000_000)
    t1 = time.perf_counter()
    with gb.Device(limit) as d2:
        t2 = time.perf_counter()
        r = gb.drain_pool(d2, pool).as_dict()
        t3 = time.perf_counter()
        hb, db = d2.io_bytes()
    t4 = time.perf_counter()
    pool.close(unlink=False)
    m = gd.merge([r])
    t5 = time.perf_counter()
    print(f"pool {t1-t0:.4f} open {t2-t1:.4f} drain {t3-t2:.4f} close {t4-t3:.4f} merge {t5-t4:.4f} total {t5-t0:.4f}", flush=True)
