"""Bounds probe of the large-prime row walk (compute-sanitizer is closed on
the GPU pool): run with the GB_LS_BOUNDS + GB_STATS variant
(tools/variants.sh bounds "" "-DGB_STATS -DGB_LS_BOUNDS") through
GB_TOOLS_LIB_OVERRIDE=1 GB_LIB_PATH=build/variants/bounds/libgoldbach_b200.so.
Every k_large_rows RED outside its slot's bitmask is counted (stat 7) and
dropped; the count must be 0 and the records must equal the default build's."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2603_07850_b200 as gb

TOP = (1 << 64) - 2
cases = [  # (start, end, segment evens)
    (4 * 10**18, 4 * 10**18 + 10**11, 200_000_000),          # C5 window, 8-slot batches
    (4 * 10**18, 4 * 10**18 + 16 * 4_000_000 - 2, 2_000_000),  # small segments, several slots
    (TOP - 3 * 10**10, TOP, 200_000_000),                      # up to the 2^64 ceiling
    (TOP - 40_000_000, TOP, 1_000_000),                         # ceiling, 20 small slots
]
v = (C.c_uint64 * 8)()
for a, b, seg in cases:
    with gb.Device(b, max_seg_evens=seg) as dev:
        gb.lib().gb_debug_stats(v, 1)
        r = gb.drain_pool(dev, gb.Pool(a, b, seg)).as_dict()
        gb.lib().gb_debug_stats(v, 1)
        print(f"[{a}, {b}] seg={seg} oob_reds={v[7]} sum={r['sum_pmin']} hash={r['pos_hash']} "
              f"max={r['max_p']}@{r['max_n']} segments={r['segments']} unverified={r['unverified']}", flush=True)
