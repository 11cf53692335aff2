"""The goldbach CLI (paper_2603_07850_b200/bin/goldbach) against the
reference CLI (oracle/_ref/goldbach_ref, built from /root/reference):
flag grammar, validation messages and exit codes (cli.cpp:140-224,
tools/main.cpp:8-24) on CPU; full runs, JSON keys and the inject-fail
exit-2 path (cli.cpp:305-334, acceptance c1/c8/c9) on the GPU."""
import json
import os
import subprocess

import pytest

from conftest import ROOT

OURS = os.path.join(ROOT, "paper_2603_07850_b200", "bin", "goldbach")
REF = os.path.join(ROOT, "oracle", "_ref", "goldbach_ref")

need_bins = pytest.mark.skipif(not (os.path.exists(OURS) and os.path.exists(REF)),
                               reason="CLI binaries not built")


def run(exe, *args, timeout=600):
    p = subprocess.run([exe, *args], capture_output=True, text=True, timeout=timeout)
    return p.returncode, p.stdout, p.stderr


def before_usage(err):
    return err.split("\nusage:")[0].strip()


BAD = [[], ["abc"], ["3"], ["100", "--seg-size=0"], ["100", "--seg-size=4294967296"],
       ["100", "--start=2"], ["18446744073709551616"], ["100", "--bogus"],
       ["100", "--p-small=2"], ["100", "--start=200"], ["100", "--batch-size=0"],
       ["100", "--start=abc"], ["-5"], ["100", "200"], ["100", "--inject-fail"]]


@need_bins
@pytest.mark.parametrize("args", BAD, ids=lambda a: " ".join(a) or "<none>")
def test_usage_errors_match_reference(args):
    rr, _, er = run(REF, *args)
    ro, _, eo = run(OURS, *args)
    assert rr == ro == 1
    assert before_usage(eo) == before_usage(er)


@need_bins
def test_help_exit_zero():
    assert run(OURS, "--help")[0] == 0
    assert "usage: goldbach" in run(OURS, "--help")[1]


@need_bins
def test_workers_zero_rejected():
    ro, _, eo = run(OURS, "100", "--workers=0")
    assert ro == 1 and "workers must be >= 1, or -1" in eo


@pytest.mark.gpu
@need_bins
def test_json_summary_matches_reference_1e9():
    """acceptance c1 / README.md:96-113: 1e9 -> 499,999,999 evens, 0
    unverified, max 1789 @ 721,013,438; same JSON keys in the same order
    (cli.cpp:117-134) plus the checksum fields."""
    ro, out, err = run(OURS, "1000000000", "--json", "--gpus=1")
    assert ro == 0, err
    j = json.loads(out.strip().splitlines()[-1])
    keys = ["limit", "start", "workers_used", "seg_size", "p_small", "batch_size",
            "phase2_limit", "total_evens", "unverified_total", "phase2_total", "counterexamples",
            "max_min_prime", "max_min_prime_n", "segments", "per_worker_segments",
            "wall_seconds", "verified"]
    assert [k for k in j if k in keys] == keys
    assert j["total_evens"] == 499_999_999 and j["unverified_total"] == 0
    assert (j["max_min_prime"], j["max_min_prime_n"]) == (1789, 721_013_438)
    assert j["segments"] == 3 and j["verified"] is True


@pytest.mark.gpu
@need_bins
def test_inject_fail_exit_2():
    ro, out, err = run(OURS, "100000000", "--inject-fail=60119912", "--json")
    assert ro == 2
    assert "counterexample: n = 60119912 has no prime partition" in err
    j = json.loads(out.strip().splitlines()[-1])
    assert j["counterexamples"] == [60119912] and j["verified"] is False


@pytest.mark.gpu
@need_bins
def test_split_runs_sum():
    """acceptance c8: disjoint --start ranges sum to the whole."""
    whole = json.loads(run(OURS, "2000000000", "--json")[1].strip().splitlines()[-1])
    a = json.loads(run(OURS, "1000000000", "--json")[1].strip().splitlines()[-1])
    b = json.loads(run(OURS, "2000000000", "--start=1000000002", "--json")[1]
                   .strip().splitlines()[-1])
    assert a["total_evens"] + b["total_evens"] == whole["total_evens"]
    assert max(a["max_min_prime"], b["max_min_prime"]) == whole["max_min_prime"]
    # the checksums are sums over evens, the segments a partition of the range
    M = (1 << 64) - 1
    assert (a["pmin_sum"] + b["pmin_sum"]) & M == whole["pmin_sum"]
    assert (a["pmin_hash"] + b["pmin_hash"]) & M == whole["pmin_hash"]
    assert a["segments"] + b["segments"] == whole["segments"] + 1  # 2e9 / 4e8: the cut splits one segment
    assert a["unverified_total"] + b["unverified_total"] == whole["unverified_total"] == 0
    w = max((a, b), key=lambda r: (r["max_min_prime"], -r["max_min_prime_n"]))
    assert w["max_min_prime_n"] == whole["max_min_prime_n"]


@pytest.mark.gpu
@need_bins
@pytest.mark.parametrize("k", [1, 2, 4])
def test_cli_worker_count_invariance(k):
    """acceptance c6 (acceptance.cpp:188-248): --gpus=k workers (round-robin
    over the visible GPUs, so k workers share GPU 0 on a 1-GPU box) give the
    same totals, checksums and max for every k; every worker claims work."""
    ro, out, err = run(OURS, "20000000000", "--json", f"--gpus={k}")
    assert ro == 0, err
    j = json.loads(out.strip().splitlines()[-1])
    assert j["workers_used"] == k and len(j["per_worker_segments"]) == k
    assert sum(j["per_worker_segments"]) == j["segments"] == 50
    assert j["total_evens"] == 9_999_999_999 and j["unverified_total"] == 0
    ref = json.loads(run(OURS, "20000000000", "--json", "--gpus=1")[1].strip().splitlines()[-1])
    for key in ("total_evens", "pmin_sum", "pmin_hash", "max_min_prime", "max_min_prime_n", "segments"):
        assert j[key] == ref[key], (key, j[key], ref[key])


@pytest.mark.gpu
@need_bins
def test_cli_mem_cap_rejects_before_any_claim():
    """validate_resources (cli.cpp:264-296): a cap below the per-GPU
    footprint fails with exit 1 and a ResourceError before any work."""
    ro, out, err = run(OURS, "10000000000000", "--mem-cap=1000000", "--json")
    assert ro == 1
    assert "mem" in err.lower() or "memory" in err.lower() or "exceeds" in err.lower(), err
    assert out.strip() == ""
