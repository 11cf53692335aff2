"""Mask fill of the large tile primes (k_mask_fill: every prime >= the
threshold struck once per 3-block range into the slot's large-prime bitmask,
which the fused kernel ANDs in) against the per-block row path and the
reference goldens.

The mask fill changes only WHERE a large prime's strikes come from (one
visit per 3 blocks instead of one per block), so every record must be
bit-identical to the row path and to the reference (sieve.cpp:109-126,
144-147 is the reference's own sparse-prime hit list)."""
import os

import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def _rec(dev, a, b):
    return dev.verify_segment(a, b).key()


def _open(gb, cover, **kw):
    return gb.Device(cover, **kw)


# (cover, segment a, segment evens): 1e12 / 1e13 (dense buckets, rows for the
# first multiples), C5 height and the 2^64 ceiling (sparse buckets)
CASES = [
    (10**12, 10**12 - 400_000_000 + 2, 200_000_000),
    (10**13, 9_000_000_000_004, 200_000_000),
    (4 * 10**18 + 10**11, 4 * 10**18 + 4 * 10**9, 20_000_000),
]


@pytest.mark.parametrize("cover,a,n", CASES)
def test_bucket_equals_rows(gpu, cover, a, n):
    b = a + 2 * (n - 1)
    os.environ["GB_MASK_P"] = "262145"  # on (default: off)
    try:
        dev = _open(gpu, cover)
    finally:
        del os.environ["GB_MASK_P"]
    with dev:
        info = dev.bucket_info()
        assert info["active"] == 1 and info["primes"] > 0, info
        got = _rec(dev, a, b)
        dev.set_bucket(False)
        want = _rec(dev, a, b)
        dev.set_bucket(True)
    assert got == want


@pytest.mark.parametrize("pb", ["65536", "131072", "262145", "1048576", "0"])
def test_bucket_thresholds_agree(gpu, pb):
    a, b = 10**13 - 40_000_000, 10**13
    with gpu.Device(10**13) as dev:
        want = _rec(dev, a, b)
    os.environ["GB_MASK_P"] = pb
    try:
        with gpu.Device(10**13) as dev:
            info = dev.bucket_info()
            assert info["active"] == (0 if pb == "0" else 1)
            assert _rec(dev, a, b) == want
    finally:
        del os.environ["GB_MASK_P"]


def test_bucket_ceiling_window(gpu):
    """Sparse buckets to p < 2^32 at the top of the number line."""
    w = golden("ceiling.json")
    recs = w["records"] if "records" in w else [w]
    r = recs[0]
    os.environ["GB_MASK_P"] = "262145"
    try:
        dev = gpu.Device(r.get("cover", (1 << 64) - 1))
    finally:
        del os.environ["GB_MASK_P"]
    with dev:
        assert dev.bucket_info()["active"] == 1
        got = dev.verify_segment(r["a"], r["b"]).as_dict()
    for k in ("evens", "unverified", "sum_pmin", "pos_hash", "max_p", "max_n"):
        assert got[k] == r[k], (k, got, r)


def test_reference_api_conformance_gpu(gpu):
    """The device-backed reference entry points (phase1_verify,
    verify_segment, phase2_resolve, is_prime_u64, build_base_primes,
    tiled_sieve_segment) through the reference signatures."""
    import subprocess
    from conftest import ROOT
    exe = os.path.join(ROOT, "paper_2603_07850_b200", "bin", "ref_api_conformance")
    out = subprocess.run([exe, "--gpu"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr[-2000:]
    assert "conformance ok" in out.stdout


@pytest.mark.parametrize("cover,a,n", CASES + [(10**12, 10**12 - 2 * 3_000_000 + 2, 3_000_000)])
def test_pair_mode_equals_default(gpu, cover, a, n):
    """k_verify_pair (2-CTA clusters sharing the single-strike rows through
    DSMEM, GB_PAIR=1) against the default kernel; the last case has an odd
    block count (4 blocks + a partial one) so one CTA of the last pair has
    no block of its own."""
    b = a + 2 * (n - 1)
    with _open(gpu, cover) as dev:
        want = _rec(dev, a, b)
    os.environ["GB_PAIR"] = "1"
    try:
        dev = _open(gpu, cover)
    finally:
        del os.environ["GB_PAIR"]
    with dev:
        assert _rec(dev, a, b) == want
