"""Small runs for compute-sanitizer (memcheck / racecheck): the fused kernel
on the row path, with the mask fill, and on the large-prime bitmask path
(one segment: k_large_rows row 0 only; large8: 8 consecutive segments in
flight, so batches of several slots take both k_large_rows launches)."""
import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2603_07850_b200 as gb
mode = sys.argv[1] if len(sys.argv) > 1 else "rows"
if mode == "mask":
    os.environ["GB_MASK_P"] = "262145"
if mode == "large8":
    a = 4 * 10**18
    with gb.Device(a + 10**11, max_seg_evens=2_000_000) as dev:
        pool = gb.Pool(a, a + 16 * 4_000_000 - 2, 2_000_000)
        r = gb.drain_pool(dev, pool)
        print(mode, dev.bucket_info(), r.as_dict())
    sys.exit(0)
cover, a = {"rows": (10**12, 10**12 - 6_000_000), "mask": (10**13, 10**13 - 6_000_000),
            "large": (4 * 10**18 + 10**11, 4 * 10**18)}[mode]
with gb.Device(cover, max_seg_evens=2_000_000) as dev:
    r = dev.verify_segment(a, a + 2 * (2_000_000 - 1))
    print(mode, dev.bucket_info(), r.as_dict())
