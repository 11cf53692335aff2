#!/usr/bin/env python3
"""bench.py -- throughput of the B200 Goldbach verifier (north star: "even n
verified/sec; wall time to 1e12 (1 GPU) and 1e13 at 1/2/4/8 B200").

One STEP = one full verification pass over the workload's range of evens
through the work-stealing pool: every rank drains ONE shared segment cursor
(claim_next semantics, proj/src/pool.cpp:24-31) on its own GPU, then the
per-rank records are merged with one all-gather (pool.cpp:159-174).  The
default workload is C3 = [4, 1e12] (BASELINE.json configs[2], the paper's
single-GPU 36.5 s headline); `--limit 1e13` is C4.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--limit L] [--impl ours|reference]

`value`  : evens/s over the K device-timed steps (CUDA events on the
           library's own streams, device drained on both sides, max over
           ranks), device handle and tables resident.
`e2e`    : the same metric through the public API a user calls, per step:
           gb_open (K1 base primes on the device) + pool drain + records
           back to the host + close + the final all-gather; h2d/d2h bytes
           are the job descriptors and records that cross PCIe.
`roofline`: the fused sieve+check kernel (k_verify_ws), algorithmic
           shared-memory bytes per launch (SURVEY.md sec. 8d frozen formula
           B(N) = 4 S(sqrt N) + 16 W64(N) + 0.25 B per even) / its average
           launch duration, against the shared-memory bandwidth measured live
           on this GPU by gb_smem_peak.
`cpu_baseline`: the UNMODIFIED reference CLI (oracle/_ref/goldbach_ref, built
           from /root/reference by oracle/build_ref.sh) on a bounded sample of
           the same workload on this host's cores.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SPAN_DEFAULT = 200_000_000
METRIC = "even n verified/sec"
UNIT = "evens/s"

# algorithmic shared-memory bytes per even n,
# B(N) = 4*S(sqrt N) + 16*W64(N) + 0.25, frozen at these range tops
# (interpolated linearly in log10 N in between).
ALG_BYTES_PER_EVEN = [(1e8, 24.7), (1e10, 26.6), (1e12, 28.3), (1e13, 29.2), (4e18, 34.4)]


def alg_bytes_per_even(limit: float) -> float:
    x = math.log10(max(limit, 1e8))
    pts = [(math.log10(n), b) for n, b in ALG_BYTES_PER_EVEN]
    if x >= pts[-1][0]:
        return pts[-1][1]
    for (x0, b0), (x1, b1) in zip(pts, pts[1:]):
        if x0 <= x <= x1:
            return b0 + (b1 - b0) * (x - x0) / (x1 - x0)
    return pts[0][1]


def load_json(path):
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return None


# --------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi equivalent via NVML, sampled every 100 ms in a thread."""

    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
        "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
        "display_clock_setting": 0x100,
    }

    def __init__(self, index: int):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._ok = True
        except Exception as e:  # no NVML: report it rather than invent clocks
            self.error = repr(e)
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for name, bit in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        if self._ok:
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._ok:
            self._t.join()

    def summary(self):
        if not self._ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# --------------------------------------------------------------- distributed
class Dist:
    def __init__(self, n_gpus: int):
        self.rank = int(os.environ.get("RANK", "0"))
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.local_rank = int(os.environ.get("LOCAL_RANK", str(self.rank)))
        if self.world != n_gpus and self.world > 1:
            raise SystemExit(f"--gpus {n_gpus} but WORLD_SIZE={self.world}")
        self.tdev = None
        # GB_BENCH_BACKEND=gloo + GB_BENCH_SHARE_GPU=1: a box with fewer GPUs
        # than ranks runs the multi-rank path (shared cursor, all-gather
        # merge, max-over-ranks timing) with every rank on GPU 0 -- a
        # correctness check of that path, not a scaling measurement
        self.backend = os.environ.get("GB_BENCH_BACKEND", "nccl")
        self.gpu = self.local_rank
        if os.environ.get("GB_BENCH_SHARE_GPU") == "1":
            import torch
            self.gpu = self.local_rank % max(torch.cuda.device_count(), 1)
        if self.world > 1:
            import torch
            import torch.distributed as dist
            torch.cuda.set_device(self.gpu)
            if self.backend == "nccl":
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.gpu))
                self.tdev = torch.device("cuda", self.gpu)
            else:
                dist.init_process_group(self.backend)
                self.tdev = torch.device("cpu")
        self.tag = os.environ.get("MASTER_PORT", "0")

    def barrier(self):
        if self.world > 1:
            import torch.distributed as dist
            if self.backend == "nccl":
                dist.barrier(device_ids=[self.gpu])
            else:
                dist.barrier()

    def max(self, x):
        if self.world == 1:
            return x
        from paper_2603_07850_b200 import dist as gd
        return gd.max_over_ranks(x, device=self.tdev)

    def sum(self, x):
        if self.world == 1:
            return x
        from paper_2603_07850_b200 import dist as gd
        return gd.sum_over_ranks(x, device=self.tdev)

    def merge(self, res: dict) -> dict:
        from paper_2603_07850_b200 import dist as gd
        if self.world == 1:
            return gd.merge([res])
        return gd.allgather_merge(res, device=self.tdev)

    def close(self):
        if self.world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


def make_pool(gb, D: Dist, args, name: str):
    """One shared cursor for every rank (rank 0 creates it)."""
    if D.world == 1:
        return gb.Pool(args.start, args.limit, args.seg_size)
    shm = f"/gb_bench_{D.tag}_{name}"
    pool = None
    if D.rank == 0:
        pool = gb.Pool(args.start, args.limit, args.seg_size, shm_name=shm, create=True)
    D.barrier()
    if D.rank != 0:
        pool = gb.Pool(args.start, args.limit, args.seg_size, shm_name=shm, create=False)
    return pool


def release_pool(D: Dist, pool):
    D.barrier()  # everyone is done with the cursor
    pool.close(unlink=(D.rank == 0))


# --------------------------------------------------------------- CPU legs
def cpu_reference_sample(args, cores: int, target_s: float = 15.0):
    """Times the reference CPU implementation on a bounded sample of the
    workload: 2 segments per host thread taken from the middle of the range.
    oracle/_ref/goldbach_ref (kind "reference") when it was built, else the
    oracle's C port (kind "port")."""
    span = 2 * args.seg_size
    n_total = (args.limit - args.start) // span + 1
    n_seg = max(1, min(n_total, 2 * cores))
    k0 = max(0, min(n_total - n_seg, n_total // 2))
    s = args.start + k0 * span
    lim = min(args.limit, s + n_seg * span - 2)
    sample = (f"segments {k0}..{k0 + n_seg - 1} of the workload: evens [{s}, {lim}] "
              f"({n_seg} x {args.seg_size} evens), {cores} threads")
    ref_bin = os.path.join(ROOT, "oracle", "_ref", "goldbach_ref")
    if os.path.exists(ref_bin):
        t0 = time.perf_counter()
        out = subprocess.run([ref_bin, f"--start={s}", f"--workers={cores}", "--json",
                              f"--seg-size={args.seg_size}", f"--p-small={args.p_small}", str(lim)],
                             capture_output=True, text=True, timeout=1800)
        wall = time.perf_counter() - t0
        if out.returncode != 0:
            raise RuntimeError(f"goldbach_ref failed: {out.stderr[-400:]}")
        j = json.loads(out.stdout.strip().splitlines()[-1])
        evens, secs = j["total_evens"], j["wall_seconds"]
        return {"value": evens / secs, "unit": UNIT, "cores": cores, "kind": "reference",
                "sample": sample + f"; reference wall_seconds {secs:.2f} s (tables excluded, "
                                   f"as cli.cpp reports), process {wall:.2f} s",
                "evens": evens, "seconds": secs, "max_p": j["max_min_prime"],
                "max_n": j["max_min_prime_n"]}
    import oracle
    t0 = time.perf_counter()
    rec, segs = oracle.verify_range(s, lim, args.seg_size, cover=lim, p_small=args.p_small,
                                    threads=cores)
    secs = time.perf_counter() - t0
    return {"value": rec.evens_checked / secs, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": sample + f"; oracle C port {secs:.2f} s", "evens": rec.evens_checked,
            "seconds": secs}


def cli_process_time(args):
    """Wall time of one `bin/goldbach LIMIT --gpus=1 --json` process (the
    reference's user-facing command, cli.cpp:298-334), measured twice; its
    JSON summary must agree with the device-timed passes."""
    exe = os.path.join(ROOT, "paper_2603_07850_b200", "bin", "goldbach")
    if not os.path.exists(exe):
        return None
    walls, j = [], None
    for _ in range(2):
        t0 = time.perf_counter()
        out = subprocess.run([exe, str(args.limit), "--gpus=1", "--json", f"--seg-size={args.seg_size}",
                              f"--p-small={args.p_small}"], capture_output=True, text=True, timeout=900)
        walls.append(time.perf_counter() - t0)
        if out.returncode != 0:
            return {"error": out.stderr[-300:]}
        j = json.loads(out.stdout.strip().splitlines()[-1])
    return {"process_s": min(walls), "runs_s": walls, "wall_seconds_reported": j.get("wall_seconds"),
            "max_min_prime": j.get("max_min_prime"), "max_min_prime_n": j.get("max_min_prime_n"),
            "total_evens": j.get("total_evens")}


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference_arm(args, D: Dist):
    """--impl reference: the reference's own CPU path on this host."""
    if D.rank != 0:
        return
    cores = host_cores()
    for _ in range(args.warmup if args.ref_warmup else 0):
        cpu_reference_sample(args, cores)
    vals, secs = [], 0.0
    last = None
    for _ in range(args.steps):
        last = cpu_reference_sample(args, cores)
        vals.append(last["value"])
        secs += last["seconds"]
    value = args.steps * last["evens"] / secs
    cb = {k: last[k] for k in ("unit", "cores", "kind", "sample")}
    cb["value"] = value
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup if args.ref_warmup else 0,
        "ms_per_step": 1e3 * secs / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic (deterministic integer range)",
        "config": config_of(args, D), "cpu_baseline": cb,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "each step is a bounded sample of the workload (the whole range is ~"
                f"{(args.limit - args.start) / 2 / value / 3600:.1f} h on these cores)",
    }
    print(json.dumps(line), flush=True)


def config_of(args, D):
    return {"workload": args.workload, "range": [args.start, args.limit],
            "seg_size": args.seg_size, "p_small": args.p_small,
            "segments": (args.limit - args.start) // (2 * args.seg_size) + 1,
            "parallelism": f"work-stealing x{D.world}",
            "l2": "flushed (256 MiB write) before every timed step; working set per step is "
                  "~0.3 MB of tables, inputs are integer ranges"}


# --------------------------------------------------------------- main arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--limit", type=float, default=1e12)
    ap.add_argument("--start", type=int, default=4)
    ap.add_argument("--seg-size", type=int, default=SPAN_DEFAULT)
    ap.add_argument("--p-small", type=int, default=1_000_000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cli", action="store_true", help="skip the CLI process timing")
    ap.add_argument("--ref-warmup", action="store_true",
                    help="also run the warm-up steps in the reference arm")
    args = ap.parse_args()
    args.limit = int(args.limit)
    args.limit -= args.limit & 1
    args.workload = {10**12: "C3: verify all even n <= 1e12 (1 GPU headline)",
                     10**13: "C4: verify all even n <= 1e13 (work-stealing)",
                     10**10: "C2: verify all even n <= 1e10",
                     10**8: "C1: verify all even n <= 1e8"}.get(
        args.limit if args.start == 4 else -1, f"evens [{args.start}, {args.limit}]")

    D = Dist(args.gpus)
    if args.impl == "reference":
        run_reference_arm(args, D)
        D.close()
        return

    import paper_2603_07850_b200 as gb

    # cold open: the first handle of this process (CUDA context, module,
    # K1 base primes, batch buffers) -- the init cost a CLI run pays
    t_open = time.perf_counter()
    dev = gb.Device(args.limit, p_small=args.p_small, device=D.gpu,
                    max_seg_evens=args.seg_size)
    cold_open_s = D.max(time.perf_counter() - t_open)
    total_evens = (args.limit - args.start) // 2 + 1

    def pass_once(name, timed):
        pool = make_pool(gb, D, args, name)
        D.barrier()
        dev.timer_start()
        res = gb.drain_pool(dev, pool)
        ms = dev.timer_stop()
        release_pool(D, pool)
        return ms, res.as_dict()

    # ---- warm-up (also checks the whole range is covered exactly once)
    for w in range(args.warmup):
        dev.flush_l2()
        _, r = pass_once(f"w{w}", False)
        m = D.merge(r)
        if m["evens"] != total_evens or m["unverified"] or m["n_ce"]:
            raise SystemExit(f"warm-up pass wrong: {m}")

    # ---- timed steps (device time, max over ranks)
    smem_peak = dev.smem_peak()
    l0 = dev.launch_count()
    dev.kernel_times(reset=True)
    step_ms, merged = [], None
    with ClockSampler(D.gpu) as clk:
        for k in range(args.steps):
            dev.flush_l2()
            dev.set_timing(1)
            ms, r = pass_once(f"t{k}", True)
            dev.set_timing(0)
            step_ms.append(D.max(ms))
            merged = D.merge(r)
            if merged["evens"] != total_evens:
                raise SystemExit(f"timed pass covered {merged['evens']} evens, want {total_evens}")
    launches = D.sum(dev.launch_count() - l0)
    kms, kl = dev.kernel_times(reset=True)
    my_evens = r["evens"]  # this rank's share of the last step
    total_ms = sum(step_ms)
    value = args.steps * total_evens / (total_ms / 1e3)

    # ---- roofline of the fused kernel (this rank's launches, all K steps)
    verify_ms, verify_launches = kms[0], kl[0]
    bpe = alg_bytes_per_even(args.limit)
    evens_timed_rank = my_evens * args.steps
    per_launch_bytes = bpe * evens_timed_rank / max(verify_launches, 1)
    avg_launch_s = verify_ms / 1e3 / max(verify_launches, 1)
    achieved_gbs = per_launch_bytes / avg_launch_s / 1e9 if avg_launch_s > 0 else None
    peak_gbs = smem_peak / 1e9
    prof = load_json(os.path.join(ROOT, "profiles", "ncu_verify_summary.json")) or {}
    prof_w = prof.get(str(args.limit)) or {}
    # DRAM bytes of the captured launch, scaled per even to this run's launches
    per_even = prof_w.get("dram_bytes_per_even")
    traffic = per_even * evens_timed_rank / max(verify_launches, 1) if per_even else None
    peaks = load_json(os.path.join(ROOT, "MEASURED_PEAKS.json")) or {}
    roofline = {
        "bound": "smem", "kernel": "k_verify_ws (fused K2 sieve + K3 check, warp-specialised)",
        "achieved": achieved_gbs, "peak": peak_gbs, "unit": "GB/s",
        "frac": (achieved_gbs / peak_gbs) if achieved_gbs and peak_gbs else None,
        "traffic": traffic,
        "peak_source": "measured live on this GPU (gb_smem_peak: conflict-free LDS.128, "
                       "2 CTAs x 512 threads per SM)",
        "alg_bytes_per_even": bpe, "evens_per_launch": evens_timed_rank / max(verify_launches, 1),
        "alg_bytes_per_launch": per_launch_bytes, "avg_launch_ms": avg_launch_s * 1e3,
        "launches": verify_launches,
        "share_of_step": (verify_ms / sum(step_ms)) if D.world == 1 else None,
        "hbm": {"traffic_per_launch": traffic,
                "gbs": (traffic / avg_launch_s / 1e9) if traffic and avg_launch_s else None,
                "peak_gbs": peaks.get("hbm_gbs"), "peak_source": "MEASURED_PEAKS.json hbm_gbs"},
        "ncu_profile": prof_w.get("source"),
        # the kernel's own ceilings from that capture: the formula frac above
        # counts reference-algorithm bytes; these are the pipes it actually fills
        "ncu_pipes_pct": prof_w.get("pipes_pct"),
    }

    # ---- e2e through the public API, host <-> device copies included (one
    # untimed pass first: a second handle's first open allocates its pinned
    # and device buffers, later opens reuse them from the process arena)
    e2e_s, h2d, d2h = [], 0, 0
    for k in range(-1, args.steps):
        D.barrier()
        t0 = time.perf_counter()
        pool = make_pool(gb, D, args, f"e{k}")
        with gb.Device(args.limit, p_small=args.p_small, device=D.gpu,
                       max_seg_evens=args.seg_size) as d2:
            r = gb.drain_pool(d2, pool).as_dict()
            hb, db = d2.io_bytes()
        release_pool(D, pool)
        m = D.merge(r)
        dt = D.max(time.perf_counter() - t0)
        if m != merged:
            raise SystemExit(f"e2e result differs from the device-timed pass: {m} vs {merged}")
        h2d, d2h = D.sum(hb), D.sum(db)
        if k >= 0:
            e2e_s.append(dt)
    e2e_value = args.steps * total_evens / sum(e2e_s)

    # warm open (context up, arena reused): what a second handle costs
    t_open = time.perf_counter()
    gb.Device(args.limit, p_small=args.p_small, device=D.gpu, max_seg_evens=args.seg_size).close()
    warm_open_s = D.max(time.perf_counter() - t_open)
    # the whole CLI process (bin/goldbach LIMIT --gpus=1 --json): cold
    # process start, context, tables, drain, summary -- the user's wall time
    cli = None
    if D.world == 1 and args.start == 4 and not args.no_cli:
        cli = cli_process_time(args)

    cpu = None
    if D.world == 1 and not args.no_cpu_baseline:
        cpu = cpu_reference_sample(args, host_cores())

    if D.rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": D.world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "u64", "data": "synthetic (deterministic integer range; no dataset)",
            "config": config_of(args, D),
            "result": {"evens": merged["evens"], "unverified": merged["unverified"],
                       "phase2": merged["phase2"], "sum_pmin": merged["sum_pmin"],
                       "pos_hash": merged["pos_hash"], "max_p": merged["max_p"],
                       "max_n": merged["max_n"], "counterexamples": merged["n_ce"],
                       "segments": merged["segments"]},
            "wall_seconds_per_pass": total_ms / args.steps / 1e3,
            "paper_rtx5090_seconds": {10**12: 36.5116, 10**13: 133.5}.get(args.limit),
            "paper_note": {10**12: "1x RTX 5090 (PAPER.md:454)",
                           10**13: "4x RTX 5090 (PAPER.md:455)"}.get(args.limit),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "seconds_per_step": sum(e2e_s) / args.steps,
                    "step_seconds": e2e_s},
            "init": {"cold_open_s": cold_open_s, "warm_open_s": warm_open_s,
                     "note": "gb_open on the bench GPU: first handle of the process (CUDA "
                             "context, module, device K1 tables, buffers) and a second one"},
            "cli_process_s": cli,
            "gpu_launches": launches,
            "roofline": roofline,
            "cpu_baseline": ({k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")}
                             if cpu else None),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    dev.close()
    D.close()


if __name__ == "__main__":
    main()
