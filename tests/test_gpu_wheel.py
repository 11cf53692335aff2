"""Device parity on the cases the wheel-6 tile layout makes special (see
DESIGN.md sec. 3): segment starts in every residue class mod 6, segments
that end in partial blocks / partial class words, tiny segments, windows
near the start of the number line (low-window fix-up) with and without
large primes in the global bitmask, and p_small around the fast-path bound.
The checker is the CPU oracle (oracle/oracle.c, pinned against the
reference's goldens by tests/test_oracle_golden.py)."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

E6 = 782304  # evens per wheel-6 block (gb_device.cuh)


def same(got, want):
    g, w = got.as_dict(), want.as_dict()
    for k in ("a", "b", "evens", "unverified", "phase2", "sum_pmin", "pos_hash", "max_p",
              "max_n", "n_ce", "ce"):
        assert g[k] == w[k], (k, g, w)


@pytest.mark.parametrize("base", [10**9, 10**12 + 2, 10**16 + 4])
def test_starts_in_every_class_and_partial_blocks(gpu, base):
    cover = base + 2 * (2 * E6 + 200)
    with gpu.Device(cover) as dev:
        for r in (0, 2, 4):
            a = base - base % 6 + r
            if a < base:
                a += 6
            # 1e16: base primes past 2^22, so the global large-prime bitmask is on
            for n_evens in (2 * E6 - 1, 2 * E6, 2 * E6 + 1, 2 * E6 + 33, E6 // 3 + 5):
                b = a + 2 * (n_evens - 1)
                same(dev.verify_segment(a, b), oracle.verify_segment(a, b, cover=cover))


@pytest.mark.parametrize("base", [4, 6, 8, 10, 8190, 8194, 8196, 8198, 10**7, 10**12])
def test_tiny_segments(gpu, base):
    cover = base + 100
    with gpu.Device(cover) as dev:
        for n_evens in (1, 2, 3, 4, 31, 32, 33):
            b = base + 2 * (n_evens - 1)
            same(dev.verify_segment(base, b), oracle.verify_segment(base, b, cover=cover))


def test_per_even_pmin_across_classes(gpu):
    # per-n minimal p straight from the device (PMIN kernel) vs the oracle
    for a in (10**6 + 2, 10**10 + 4, 10**13):
        b = a + 2 * (E6 + 1000)
        with gpu.Device(b) as dev:
            got = dev.phase1_pmin(a, b)
        want = np.array(oracle.phase1_pmin(a, b, cover=b), dtype=np.uint64)
        bad = np.nonzero(got != want)[0]
        assert len(bad) == 0, (a, bad[:5], got[bad[:5]], want[bad[:5]])


@pytest.mark.parametrize("cover", [10**8, 2 * 10**13])
def test_low_windows(gpu, cover):
    # the first blocks of the number line: q <= 1 cleared, base primes in the
    # window restored; with cover 2e13 the base primes exceed 2^22, so the
    # global large-prime bitmask strikes these windows too
    with gpu.Device(cover) as dev:
        for a, b in ((4, 2 * 3 * E6), (2 * E6 - 40, 2 * E6 + 40), (1_564_604, 1_564_700)):
            same(dev.verify_segment(a, b), oracle.verify_segment(a, b, cover=cover))


@pytest.mark.parametrize("p_small", [3, 5, 131, 211, 223, 257, 263, 419, 421, 8191, 8193, 8209])
def test_p_small_around_the_fast_path(gpu, p_small):
    a, b = 10**9, 10**9 + 2 * 100_000
    with gpu.Device(b, p_small=p_small) as dev:
        same(dev.verify_segment(a, b), oracle.verify_segment(a, b, cover=b, p_small=p_small))


def test_reference_known_answers(gpu):
    # [4, 1e4]: 4,999 evens, max 173 @ 7426 (test_verifier.cpp:265-282);
    # p_min on [4, 20] = {2,3,3,3,5,3,3,5,3}, max 5 @ 12 (:59-73);
    # pi(1e9) = 50,847,534 (test_sieve.cpp:188-200)
    with gpu.Device(10**4) as dev:
        r = dev.verify_segment(4, 10**4).as_dict()
        assert (r["evens"], r["max_p"], r["max_n"], r["unverified"]) == (4_999, 173, 7426, 0)
        assert [int(x) for x in dev.phase1_pmin(4, 20)] == [2, 3, 3, 3, 5, 3, 3, 5, 3]
    with gpu.Device(10**9) as dev:
        assert len(dev.primes_upto(10**9)) == 50_847_534 - 1  # odd primes (2 excluded)


def test_pmin_window_above_1e12(gpu):
    # per-n p_min on [1e12, 1e12 + 400] (test_verifier.cpp:330-349) vs the oracle
    a, b = 10**12, 10**12 + 400
    with gpu.Device(b) as dev:
        got = dev.phase1_pmin(a, b)
    want = np.array(oracle.phase1_pmin(a, b, cover=b), dtype=np.uint64)
    assert (got == want).all()


def test_large_prime_batches_out_of_order(gpu):
    # base primes past 2^22, so k_large_strike runs; one batch holds pieces
    # above, below and far from its first slot (the incremental first-multiple
    # path applies only to slots 0 <= d < 2^32 wheel steps above slot 0), plus
    # neighbours 2 * E6 apart (the incremental path)
    cover = 4 * 10**16
    base = 10**16
    n_ev = E6 // 2 + 7
    starts = [base + 2 * E6 * 4, base, base + 2 * E6 * 8, 3 * 10**16 + 2, base + 2 * E6 * 9,
              base + 6 * 10**15 + 4, base + 2 * E6 * 4 + 6, 2 * 10**13 + 2]
    with gpu.Device(cover) as dev:
        for a in starts:
            dev.submit(a, a + 2 * (n_ev - 1), tag=a)
        got = {}
        for _ in starts:
            rec, tag = dev.wait()
            got[tag] = rec
    for a in starts:
        same(got[a], oracle.verify_segment(a, a + 2 * (n_ev - 1), cover=cover))
