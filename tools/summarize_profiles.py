#!/usr/bin/env python3
"""Turn a gpurun_out/ capture into the tracked summaries under profiles/.

    python tools/summarize_profiles.py <tag> [--rep gpurun_out/prof_verify.ncu-rep]
        [--launches gpurun_out/launches_bench.csv ...] [--limit 1e12] [--evens-per-launch N]

Writes profiles/<tag>_launches.txt (per-kernel share of the launch list),
profiles/<tag>_ncu_verify.txt (shared-memory / pipe / DRAM metrics of the
fused kernel + the hottest SASS basic blocks) and merges the DRAM traffic
per launch into profiles/ncu_verify_summary.json, which bench.py reads for
roofline.traffic.
"""
import argparse
import collections
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

METRICS = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__registers_per_thread",
    "launch__occupancy_limit_shared_mem", "sm__cycles_elapsed.avg.per_second",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__bytes.sum.per_second",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum",
    "lts__t_bytes.sum", "lts__t_sectors_op_read.sum", "lts__t_sectors_op_write.sum",
    "lts__t_sectors_op_red.sum", "lts__t_sectors_op_atom.sum", "lts__t_sector_hit_rate.pct",
]


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True)
    return list(csv.reader(io.StringIO(out.stdout)))


def launches_summary(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        k = r[ki].split("(")[0]
        agg[k][0] += 1
        agg[k][1] += float(r[vi].replace(",", ""))
    tot = sum(v[1] for v in agg.values()) or 1.0
    lines = [f"# {os.path.basename(path)}: ncu --metrics gpu__time_duration.sum --clock-control none",
             f"# total {tot / 1e6:.3f} ms over {sum(v[0] for v in agg.values())} launches "
             "(serialised, cold-cache: compare shares)",
             f"{'kernel':42s} {'launches':>8s} {'total_ms':>10s} {'share':>7s} {'avg_us':>10s}"]
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{k:42s} {v[0]:8d} {v[1] / 1e6:10.3f} {100 * v[1] / tot:6.1f}% {v[1] / v[0] / 1e3:10.1f}")
    return "\n".join(lines) + "\n"


def sass_blocks(rep, top=25):
    rows = ncu_csv(rep, "--page", "source", "--print-source", "sass")
    hdr = rows[1]
    ie = hdr.index("Instructions Executed")
    data = [(r[1].strip(), int(r[ie] or 0)) for r in rows[2:] if len(r) > ie]
    blocks, cur = [], None
    for i, (s, c) in enumerate(data):
        if cur and c == cur[1]:
            cur[2] += 1
            cur[3].append(s)
        else:
            cur = [i, c, 1, [s]]
            blocks.append(cur)
    tot = sum(b[1] * b[2] for b in blocks) or 1
    out = [f"# hottest SASS basic blocks (warp-instructions executed; total {tot:,})"]
    for b in sorted(blocks, key=lambda b: -b[1] * b[2])[:top]:
        out.append(f"sass#{b[0]:5d} x{b[1]:>10,} ninst {b[2]:3d} = {b[1] * b[2] / 1e6:7.1f}M "
                   f"({100 * b[1] * b[2] / tot:4.1f}%)  {b[3][0][:48]} .. {b[3][-1][:36]}")
    return "\n".join(out) + "\n", tot


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("--rep", default=os.path.join(ROOT, "gpurun_out", "prof_verify.ncu-rep"))
    ap.add_argument("--launches", nargs="*", default=[])
    ap.add_argument("--limit", type=float, default=1e12)
    ap.add_argument("--evens-per-launch", type=float, default=None)
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)
    if a.launches:
        with open(os.path.join(PROF, f"{a.tag}_launches.txt"), "w") as f:
            for p in a.launches:
                f.write(launches_summary(p) + "\n")
    if os.path.exists(a.rep):
        rows = ncu_csv(a.rep, "--page", "raw")
        hdr, units, vals = rows[0], rows[1], rows[2]
        m = {h: (vals[i], units[i]) for i, h in enumerate(hdr)}
        txt = [f"# ncu --set full --clock-control none --import-source on -k regex:k_verify "
               f"({os.path.basename(a.rep)}) {a.note}"]
        for k in METRICS:
            if k in m:
                txt.append(f"{k:90s} {m[k][0]:>20s} {m[k][1]}")
        blocks, tot = sass_blocks(a.rep)
        txt.append("")
        txt.append(blocks)

        def num(k):
            v, u = m[k]
            x = float(v.replace(",", ""))
            return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-6,
                        "msecond": 1e-3, "nsecond": 1e-9, "us": 1e-6, "ms": 1e-3,
                    "ns": 1e-9, "s": 1.0}.get(u, 1)
        dram = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
        dur = num("gpu__time_duration.sum")
        txt.append(f"dram bytes per launch {dram:.4g}  duration {dur * 1e3:.3f} ms  "
                   f"-> {dram / dur / 1e9:.2f} GB/s")
        if a.evens_per_launch:
            txt.append(f"evens per launch {a.evens_per_launch:.4g}: {dram / a.evens_per_launch:.5f} "
                       f"DRAM B/even, {tot * 32 / a.evens_per_launch:.1f} thread-instr/even")
        with open(os.path.join(PROF, f"{a.tag}_ncu_verify.txt"), "w") as f:
            f.write("\n".join(txt) + "\n")
        sp = os.path.join(PROF, "ncu_verify_summary.json")
        summ = json.load(open(sp)) if os.path.exists(sp) else {}
        key = str(int(a.limit))
        per_even = dram / a.evens_per_launch if a.evens_per_launch else None
        summ[key] = {"dram_bytes_per_launch_captured": dram, "evens_per_launch_captured": a.evens_per_launch,
                     "dram_bytes_per_even": per_even, "duration_ms_captured": dur * 1e3,
                     "pipes_pct": {"issue_active": num("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                                   "alu": num("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
                                   "smem_wavefronts": num("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
                                   "l2_hit_rate": num("lts__t_sector_hit_rate.pct")},
                     "source": f"profiles/{a.tag}_ncu_verify.txt"}
        json.dump(summ, open(sp, "w"), indent=1)
    print("ok")


if __name__ == "__main__":
    main()
