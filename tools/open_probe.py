import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
os.environ["GB_DEBUG_OPEN"] = "1"
import paper_2603_07850_b200 as gb
for cover in (10**12, 10**13, 4 * 10**18 + 10**11, 4 * 10**18 + 10**11):
    t = time.perf_counter()
    d = gb.Device(cover)
    t1 = time.perf_counter()
    d.close()
    print(f"cover {cover:.3e}: open {1e3*(t1-t):.1f} ms close {1e3*(time.perf_counter()-t1):.1f} ms", flush=True)
