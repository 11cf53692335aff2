#!/usr/bin/env python3
"""Attribute ncu warp-stall samples and executed instructions of one kernel
to source regions (the device function each SASS instruction was inlined
from, by its innermost -lineinfo line).

    python tools/ncu_regions.py REP.ncu-rep OBJ.o [--kernel k_verify_blocks]

REP must have been captured from a library built from the same sources as
OBJ (the SASS is matched by offset within the function).
"""
import argparse
import bisect
import collections
import csv
import io
import os
import re
import subprocess
import tempfile

FUNC_RE = re.compile(r"^(?:template\s*<[^>]*>\s*)?(?:__global__|__device__)[^(]*?\b(\w+)\s*\(")


def sass_rows(rep, kernel):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "-k", f"regex:{kernel}"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hdr_i]
    recs = []
    for r in rows[hdr_i + 1:]:
        if len(r) != len(hdr) or not r[0].startswith("0x"):
            continue
        recs.append(dict(zip(hdr, r)))
    return hdr, recs


def line_map(obj, kernel):
    """offset -> (file, line) for the kernel's SASS, from nvdisasm -g."""
    with tempfile.TemporaryDirectory() as td:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=td, check=True,
                       capture_output=True)
        cubins = [os.path.join(td, f) for f in os.listdir(td) if f.endswith(".cubin")]
        text = subprocess.run(["nvdisasm", "-gi", "-c", cubins[0]], capture_output=True, text=True,
                              check=True).stdout
    m = {}
    cur_fn = None
    loc = None
    fresh = True  # -gi prints the inlining chain innermost first: keep the first line
    for ln in text.splitlines():
        s = ln.strip()
        if s.startswith(".text."):
            cur_fn = s[len(".text."):].rstrip(":")
            continue
        mm = re.match(r'//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?', s)
        if mm:
            if fresh:
                loc = (os.path.basename(mm.group(1)), int(mm.group(2)))
                if mm.group(3):  # innermost line + its call site
                    loc = loc + (os.path.basename(mm.group(3)), int(mm.group(4)))
                fresh = False
            continue
        mo = re.match(r"/\*([0-9a-f]{4,})\*/", s)
        if mo:
            fresh = True
        if mo and cur_fn and kernel in cur_fn and loc:
            m.setdefault(cur_fn, {})[int(mo.group(1), 16)] = loc
    return m


def func_spans(src_dir):
    spans = {}
    for fn in os.listdir(src_dir):
        if not fn.endswith((".cu", ".cuh", ".h")):
            continue
        starts = []
        with open(os.path.join(src_dir, fn)) as f:
            for i, ln in enumerate(f, 1):
                mm = FUNC_RE.match(ln)
                if mm:
                    starts.append((i, mm.group(1)))
        spans[fn] = starts
    return spans


TINY = {"gbar", "nb_sync", "nb_arrive"}  # attribute these to their call site


def region_of(spans, loc):
    f, line = loc[0], loc[1]
    st = spans.get(f, [])
    i = bisect.bisect_right([s for s, _ in st], line) - 1
    return f"{st[i][1]}" if i >= 0 else f"{f}:?"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("obj")
    ap.add_argument("--kernel", default="k_verify_blocks")
    ap.add_argument("--variant", default="ILb0E", help="substring of the mangled kernel to match")
    ap.add_argument("--lines", action="store_true", help="also list the hottest source lines")
    a = ap.parse_args()
    hdr, recs = sass_rows(a.rep, a.kernel)
    lm = line_map(a.obj, a.kernel)
    fn = next(k for k in lm if a.variant in k)
    offs = lm[fn]
    base = int(recs[0]["Address"], 16)
    spans = func_spans(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                    "paper_2603_07850_b200", "csrc"))
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    agg = collections.defaultdict(lambda: collections.Counter())
    lines = collections.defaultdict(lambda: collections.Counter())
    tot = collections.Counter()
    for r in recs:
        off = int(r["Address"], 16) - base
        loc = offs.get(off)
        reg = region_of(spans, loc) if loc else "?"
        if loc and len(loc) > 2 and reg in TINY:
            reg = f"{reg}@{loc[3]}"
        c = agg[reg]
        samp = int(r["Warp Stall Sampling (All Samples)"] or 0)
        inst = int(r["Instructions Executed"] or 0)
        c["samples"] += samp
        c["inst"] += inst
        tot["samples"] += samp
        tot["inst"] += inst
        for h in stall_cols:
            v = int(r[h] or 0)
            c[h] += v
            tot[h] += v
        if loc:
            lines[loc[:2]]["samples"] += samp
            lines[loc[:2]]["inst"] += inst
    print(f"# {a.rep}: {tot['samples']} stall samples, {tot['inst']:,} warp-instructions")
    print(f"{'region':28s} {'samples':>8s} {'%':>6s} {'inst%':>6s}  top stalls")
    for reg, c in sorted(agg.items(), key=lambda kv: -kv[1]["samples"]):
        if c["samples"] < tot["samples"] * 0.002:
            continue
        st = sorted(((c[h], h[6:]) for h in stall_cols), reverse=True)[:4]
        sts = " ".join(f"{n}={100.0 * v / max(c['samples'], 1):.0f}%" for v, n in st if v)
        print(f"{reg:28s} {c['samples']:8d} {100.0 * c['samples'] / tot['samples']:6.1f} "
              f"{100.0 * c['inst'] / max(tot['inst'], 1):6.1f}  {sts}")
    print("overall: " + " ".join(f"{h[6:]}={100.0 * tot[h] / tot['samples']:.1f}%"
                                 for h in sorted(stall_cols, key=lambda h: -tot[h]) if tot[h]))
    if a.lines:
        print("\n# hottest source lines")
        for loc, c in sorted(lines.items(), key=lambda kv: -kv[1]["samples"])[:30]:
            print(f"{loc[0]}:{loc[1]:<5d} samples {c['samples']:7d} ({100.0 * c['samples'] / tot['samples']:.1f}%) "
                  f"inst {c['inst']:,}")


if __name__ == "__main__":
    main()
