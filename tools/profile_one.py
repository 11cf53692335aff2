"""One batch of 8 segments of 2e8 evens just below `limit` (default 1e12):
the k_verify_blocks launch to capture with ncu."""
import sys
sys.path.insert(0, '/root/repo')
import paper_2603_07850_b200 as gb
limit = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**12
nseg = int(sys.argv[2]) if len(sys.argv) > 2 else 8
dev = gb.Device(limit)
span = 400_000_000
a0 = limit - nseg * span + 2
for k in range(nseg):
    a = a0 + k * span
    dev.submit(a, min(a + span - 2, limit), k)
for k in range(nseg):
    r, _ = dev.wait()
print("ok", r.as_dict())
