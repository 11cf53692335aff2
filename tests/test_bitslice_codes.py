"""CPU checks of the bit-sliced scan generator (tools/gen_bitslice.py) that the
fused kernel's check is built from: the per-class plane codes decode back to
p, are monotone (the block max is the max code), fit the planes, and the
sum identities word_sums relies on hold (check steps 4-5)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import gen_bitslice as g  # noqa: E402


def cands(r, pmax):
    out = []
    for p in g.odd_primes(pmax):
        if p == 3:
            if r in (2, 4):
                out.append(p)
            continue
        if (r - p) % 6 in (1, 5):
            out.append(p)
    return out


def test_codes_decode_and_are_monotone():
    for r, pmax in ((0, 257), (2, 503), (4, 503)):
        ps = cands(r, pmax)
        cs = [g.class_code(r, p, "c") for p in ps]
        assert [g.code_to_p(r, c, "c") for c in cs] == ps
        assert cs == sorted(cs) and len(set(cs)) == len(cs)
        assert max(cs) < 256  # BS6_PLANES = 8


def test_sum_identity_per_class():
    # p = 3c + kf*F + ke*Z0 with (kf, ke) = (1, 1), (1, -1), (-1, 1) for r = 0, 2, 4,
    # and kf*F + ke*Z0 = sg*(g0 + 2 g1), g0 = F & ~Z0, g1 = Z0 (r = 0) -- word_sums
    kfe = {0: (1, 1), 2: (1, -1), 4: (-1, 1)}
    for r, pmax in ((0, 257), (2, 503), (4, 503)):
        kf, ke = kfe[r]
        sg = -1 if r == 4 else 1
        for p in cands(r, pmax):
            c = g.class_code(r, p, "c")
            z0 = c & 1
            assert p == 3 * c + kf + ke * z0, (r, p, c)
            g0 = 1 - z0
            g1 = z0 if r == 0 else 0
            assert kf + ke * z0 == sg * (g0 + 2 * g1), (r, p)


def test_generated_header_matches_generator():
    # the committed header is what the generator emits with its defaults
    hdr = os.path.join(g.ROOT, "paper_2603_07850_b200", "csrc", "gb_bitslice.cuh")
    text = open(hdr).read()
    assert "#define BS6_CODE 1" in text
    assert "BS6_PMAX_R0 = 211" in text and "BS6_PMAX_R24 = 419" in text
    for r, pmax in ((0, 211), (2, 419), (4, 419)):
        code, n, _, _ = g.gen_scan6(f"bs6_scan_r{r}", r, pmax, nplanes=8, nw=g.scan6_words(419), mode="c")
        assert code in text, r
