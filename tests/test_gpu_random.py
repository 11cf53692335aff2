"""Seeded random segments across magnitudes: device vs the CPU oracle.

SURVEY.md sec. 8d: random parity segments reuse the reference's seeds
(0xacce972, acceptance.cpp:89).  Starts are log-uniform in [10^3, 10^17]
(the 2^64 ceiling is covered by tests/golden/ceiling.json), lengths uniform
in [1, 400000] evens, and every segment runs at its own cover (base primes to
sqrt(b)), so every tile path -- low windows, partial blocks, every class
alignment, the large-prime bitmask above 1.76e13 -- is drawn."""
import random

import pytest

import oracle

pytestmark = pytest.mark.gpu


def _segments(seed, n):
    rng = random.Random(seed)
    out = []
    for _ in range(n):
        a = int(10 ** rng.uniform(3, 17))
        a += a & 1
        evens = rng.randint(1, 400_000)
        out.append((a, a + 2 * (evens - 1)))
    return out


@pytest.mark.parametrize("a,b", _segments(0xACCE972, 32))
def test_random_segment(gpu, a, b):
    with gpu.Device(b) as dev:
        got = dev.verify_segment(a, b).as_dict()
    want = oracle.verify_segment(a, b, cover=b).as_dict()
    for k in ("a", "b", "evens", "unverified", "phase2", "sum_pmin", "pos_hash", "max_p", "max_n", "n_ce", "ce"):
        assert got[k] == want[k], (k, got, want)
