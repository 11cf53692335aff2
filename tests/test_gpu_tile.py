"""The fused kernel's OWN sieve (K2 inside k_verify_ws), checked cell by cell.

Every other parity test sees the fused sieve only through the minimal p it
feeds the check with, and the sieve-window hook (gb_sieve_interval) runs the
K1 interval kernel.  gb_debug_tile copies the wheel-6 tile of one block right
after its sieve (presieve patterns, warp-cooperative and row strikes, the
large-prime bitmask of k_large_strike / k_mask_fill, the low-window fix-up)
and this test compares every cell q <= min(cover, b) with the oracle's
odd-only sieve of the same window (tiled_sieve_segment, sieve.cpp:91-156):
bit set <=> q prime."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def expand(words):
    """bit k of the class array (LSB-first u32 words) as a bool array"""
    return np.unpackbits(words.astype("<u4").view(np.uint8), bitorder="little").astype(bool)


def check_tile(gb, oracle, cover, a, b, block, env=None):
    old = {k: os.environ.get(k) for k in (env or {})}
    os.environ.update(env or {})
    try:
        dev = gb.Device(cover)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    with dev:
        if block < 0:  # counted from the last block of the piece
            e6 = 3 * (32 * dev.tile_words() - 1376)
            block += ((b - a) // 2 + 1 + e6 - 1) // e6
        Q, A, B = dev.debug_tile(a, b, block)
    M6 = 32 * len(A)  # cells per class array of this build
    assert Q % 6 == 1
    top = min(cover, b)
    lo = max(Q, 3) | 1
    hi = min(Q + 6 * M6, top)
    hi -= 1 - (hi & 1)
    ref_words = oracle.sieve_words(lo, hi, cover=cover)
    ref = np.unpackbits(ref_words.astype("<u8").view(np.uint8), bitorder="little").astype(bool)
    n_checked = 0
    for arr, off in ((A, 0), (B, 4)):
        got = expand(arr)
        q = Q + off + 6 * np.arange(M6, dtype=np.int64)
        ok = (q <= hi)
        want = np.zeros(M6, dtype=bool)
        inside = ok & (q >= lo)
        want[inside] = ref[(q[inside] - lo) // 2]
        bad = np.nonzero(ok & (got != want))[0]
        assert len(bad) == 0, (cover, a, block, off, bad[:5], q[bad[:5]], got[bad[:5]])
        n_checked += int(ok.sum())
    assert n_checked > 0
    return n_checked


CASES = [
    # cover, a, b, block, env
    (10**8, 4, 10**8, 0, None),                                        # low window: q <= 1, base primes restored
    (10**8, 4, 10**8, 1, None),
    (10**12, 10**12 - 400_000_000 + 2, 10**12, 0, None),             # C3 rows
    (10**12, 10**12 - 400_000_000 + 2, 10**12, -1, None),            # last block of a segment
    (10**13, 10**13 - 400_000_000 + 2, 10**13, 117, None),           # C4 heavy split
    (10**13, 10**13 - 400_000_000 + 2, 10**13, 117, {"GB_MASK_P": "262145"}),  # mask fill
    (4 * 10**18 + 10**11, 4 * 10**18, 4 * 10**18 + 400_000_000 - 2, 3, None),  # k_large_strike bitmask
]


@pytest.mark.parametrize("cover,a,b,block,env", CASES)
def test_fused_tile_matches_oracle_sieve(gpu, cover, a, b, block, env):
    import oracle
    check_tile(gpu, oracle, cover, a, b, block, env)


def test_fused_tiles_random_heights(gpu):
    """Seeded random windows (the reference's seed 0xacce972) from 1e7 to
    1e16: one piece of up to 2e8 evens, a random block of it, every cell."""
    import random
    import oracle
    rng = random.Random(0xacce972)
    for _ in range(8):
        cover = int(10 ** rng.uniform(7, 16))
        evens = rng.randint(1, 2 * 10**6)
        a = rng.randrange(4, max(6, cover - 2 * evens), 2)
        b = min(a + 2 * (evens - 1), cover - (cover & 1))
        if b < a:
            continue
        with gpu.Device(cover) as d0:
            e6 = 3 * (32 * d0.tile_words() - 1376)  # evens per block
        nblocks = ((b - a) // 2 + 1 + e6 - 1) // e6
        check_tile(gpu, oracle, cover, a, b, rng.randrange(nblocks))
