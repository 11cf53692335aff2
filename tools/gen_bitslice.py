#!/usr/bin/env python3
"""Generate paper_2603_07850_b200/csrc/gb_bitslice.cuh.

The fused kernel's check (K3) runs bit-sliced: one lane owns 32 consecutive
evens (one 32-bit word, bit i <-> even il = 32w + i) and walks the odd prime
candidates p = 3 + 2z in ascending order.  For candidate z the 32 bits
"n - p is prime" are the tile bits at cells JH + 32w + i - z, i.e. ONE funnel
shift of two tile words with a compile-time shift.  U holds the evens whose
minimal p is not yet known: U &= ~S per candidate.  This is the word-parallel
form of phase1_verify's ascending scan (reference verifier.cpp:66-88).

The minimal p of every even is recorded bit-sliced as z = (p - 3)/2 in planes
Z[b] (bit i of Z[b] = bit b of z_i).  Plane b is the union of the z-intervals
[m 2^b, (m+1) 2^b), m odd; the evens found inside one interval are
U(before its first prime) & ~U(after its last prime), so each non-empty
interval costs one LOP3 instead of one per prime.

The funnel shift of a candidate is either one SHF (ALU pipe) or, as
hi * 2^(32-sh) + umulhi(lo, 2^(32-sh)) with the power of two read from
constant memory (so ptxas cannot fold it back into SHF), two IMADs on the
FMA pipe.  The ALU pipe is the kernel's bottleneck (LOP3/SHF/ISETP all
issue there at half rate), so most candidates take the FMA form; one in
SHF_EVERY keeps SHF to balance the two pipes against issue.

Usage: python tools/gen_bitslice.py [--shf-every N]   (rewrites the header in place)
"""
import argparse
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "paper_2603_07850_b200", "csrc", "gb_bitslice.cuh")


def odd_primes(hi):
    return [p for p in range(3, hi + 1, 2) if all(p % d for d in range(3, int(p ** 0.5) + 1, 2))]


def gen_scan(name, zmax, shf_every):
    """Scan of candidates z = 0..zmax (p = 3 + 2z prime).  Tile words
    t0..tK with tK = word B (cells 32B..32B+31 of the lane's top), t(K-k) =
    word B - k."""
    zs = [(p - 3) // 2 for p in odd_primes(3 + 2 * zmax)]
    nplanes = zmax.bit_length()
    K = (zmax + 31) // 32
    args = ", ".join(f"uint32_t t{k}" for k in range(K + 1))
    L = []
    L.append(f"// candidates p = 3..{3 + 2 * zmax} ({len(zs)} odd primes); planes Z[0..{nplanes - 1}]")
    L.append(f"__device__ __forceinline__ void {name}({args}, uint32_t& U, uint32_t (&Z)[{nplanes}]) {{")
    L.append("    uint32_t S;")
    # plane interval bookkeeping: for each plane b, the open interval id and
    # its snapshot name
    open_iv = {}
    # precompute, for every plane, the last prime index of each interval
    last_in_iv = {}
    for b in range(nplanes):
        for idx, z in enumerate(zs):
            if (z >> b) & 1:
                last_in_iv[(b, z >> b)] = idx
    first_write = [True] * nplanes
    for idx, z in enumerate(zs):
        # snapshots for intervals that start at this prime
        for b in range(nplanes):
            if (z >> b) & 1 and open_iv.get(b) != (z >> b):
                open_iv[b] = z >> b
                L.append(f"    const uint32_t s{b}_{z >> b} = U;")
        k = (z + 31) // 32
        sh = (-z) % 32
        if sh == 0:
            src = f"t{K - k}"
        elif shf_every and idx % shf_every == shf_every - 1:
            src = f"__funnelshift_r(t{K - k}, t{K - k + 1}, {sh})"
        else:
            src = f"fsr_fma(t{K - k}, t{K - k + 1}, {sh})"
        L.append(f"    S = {src}; // p = {3 + 2 * z}")
        L.append("    U &= ~S;")
        for b in range(nplanes):
            if (z >> b) & 1 and last_in_iv[(b, z >> b)] == idx:
                op = "=" if first_write[b] else "|="
                first_write[b] = False
                L.append(f"    Z[{b}] {op} s{b}_{z >> b} & ~U;")
    for b in range(nplanes):
        if first_write[b]:
            L.append(f"    Z[{b}] = 0u;")
    L.append("}")
    return "\n".join(L), len(zs), nplanes, K


def scan6_words(pmax):
    """tile words per array every class scan reads (the largest g over classes)"""
    gmax = max((p + 1) // 6 for p in odd_primes(pmax))
    return gmax // 32 + 2


def class_code(r, p, mode):
    """Plane code of candidate p in class r.  mode "z": z = (p - 3)/2 (sum p =
    3 + 2z).  mode "c": c ascends in smaller steps, so the plane intervals
    are longer and fewer (fewer LOP3s per scan):
      r = 0: p = 3c + 1 + (c & 1)            (5 -> 1, 7 -> 2, 11 -> 3, ...)
      r = 2: p = 3 -> c = 1, p = 6y + 1 -> c = 2y   (p = 3c + 1 - (c & 1))
      r = 4: p = 3 -> c = 1, p = 6y - 1 -> c = 2y   (p = 3c - 1 + (c & 1))
    so p = 3c + kf F + ke Z0 with (kf, ke) = (1, 1), (1, -1), (-1, 1)."""
    if mode == "z":
        return (p - 3) // 2
    if r == 0:
        return (p - 1) // 3 if p % 6 == 1 else (p - 2) // 3
    if p == 3:
        return 1
    return 2 * ((p - 1) // 6) if r == 2 else 2 * ((p + 1) // 6)


def code_to_p(r, c, mode):
    if mode == "z":
        return 3 + 2 * c
    if r == 0:
        return 3 * c + 1 + (c & 1)
    if r == 2:
        return 3 * c + 1 - (c & 1)
    return 3 * c - 1 + (c & 1)


def gen_scan6(name, r, pmax, nplanes=None, nw=None, fma_every=0, mode="z"):
    """Wheel-6 scan for the words of evens n = r (mod 6).  The tile holds
    two arrays, A: q = Q + 6k (q = 1 mod 6) and B: q = Q + 4 + 6k (q = 5 mod 6);
    lane bit i of word w is class-r even t = 32w - delta + i, whose candidate
    p reads array cell k = t + G - g with g = (p - eps)/6 (A) or
    (p + 4 - eps)/6 (B), eps = (r - 1) mod 6.  Only candidates with n - p
    prime-capable (q = +-1 mod 6) exist for the class: r = 2 -> p = 3 (B) and
    p = 1 mod 6 (A); r = 4 -> p = 3 (A) and p = 5 mod 6 (B); r = 0 -> p = 5
    mod 6 (A) and p = 1 mod 6 (B).  a0..a2 / b0..b2 = array words WB-2..WB."""
    eps = (r - 1) % 6
    cands = []
    for p in odd_primes(pmax):
        if p == 3:
            if r == 2:
                cands.append((p, "b", (p + 4 - eps) // 6))
            elif r == 4:
                cands.append((p, "a", (p - eps) // 6))
            continue
        q = (r - p) % 6
        if q == 1:
            cands.append((p, "a", (p - eps) // 6))
        elif q == 5:
            cands.append((p, "b", (p + 4 - eps) // 6))
    zs = [class_code(r, p, mode) for p, _, _ in cands]
    assert all(code_to_p(r, z, mode) == p for (p, _, _), z in zip(cands, zs))
    assert zs == sorted(zs) and len(set(zs)) == len(zs)
    if nplanes is None:
        nplanes = max(zs).bit_length()
    assert max(zs) < (1 << nplanes)
    L = []
    what = "z = (p - 3)/2" if mode == "z" else "the class code c (class_code in tools/gen_bitslice.py)"
    L.append(f"// class r = {r}: {len(cands)} candidates p <= {pmax}; planes Z[0..{nplanes - 1}] of {what}")
    if nw is None:
        nw = scan6_words(pmax)  # words per array: WB-(nw-1) .. WB
    args = ", ".join([f"uint32_t a{k}" for k in range(nw)] + [f"uint32_t b{k}" for k in range(nw)])
    L.append(f"__device__ __forceinline__ void {name}({args}, uint32_t& U, uint32_t (&Z)[{nplanes}]) {{")
    L.append("    uint32_t S;")
    open_iv = {}
    last_in_iv = {}
    for b in range(nplanes):
        for idx, z in enumerate(zs):
            if (z >> b) & 1:
                last_in_iv[(b, z >> b)] = idx
    first_write = [True] * nplanes
    for idx, ((p, arr, g), z) in enumerate(zip(cands, zs)):
        for b in range(nplanes):
            if (z >> b) & 1 and open_iv.get(b) != (z >> b):
                open_iv[b] = z >> b
                L.append(f"    const uint32_t s{b}_{z >> b} = U;")
        k = (g + 31) // 32
        sh = (-g) % 32
        w = [f"{arr}{i}" for i in range(nw)]  # w[nw-1] = word WB
        top = nw - 1
        if sh == 0:
            src = w[top - k]
        elif fma_every and idx % fma_every == 0:
            src = f"fsr_fma({w[top - k]}, {w[top - k + 1]}, {sh})"
        else:
            src = f"__funnelshift_r({w[top - k]}, {w[top - k + 1]}, {sh})"
        L.append(f"    S = {src}; // p = {p}")
        L.append("    U &= ~S;")
        for b in range(nplanes):
            if (z >> b) & 1 and last_in_iv[(b, z >> b)] == idx:
                op = "=" if first_write[b] else "|="
                first_write[b] = False
                L.append(f"    Z[{b}] {op} s{b}_{z >> b} & ~U;")
    for b in range(nplanes):
        if first_write[b]:
            L.append(f"    Z[{b}] = 0u;")
    L.append("}")
    return "\n".join(L), len(cands), nplanes, nw


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shf-every", type=int, default=1)
    ap.add_argument("--pbs6", type=int, default=385, help="largest bit-sliced candidate (wheel-6 scans)")
    ap.add_argument("--pbs-r0", type=int, default=211, help="class-0 bound (0: --pbs6)")
    ap.add_argument("--fma-every", type=int, default=0,
                    help="every N-th candidate's funnel shift on the FMA pipe (0: none)")
    ap.add_argument("--pbs-r24", type=int, default=419, help="classes 2/4 bound (0: --pbs6)")
    ap.add_argument("--code", choices=["z", "c"], default="c",
                    help="plane code: z = (p-3)/2, or the per-class code c (fewer plane intervals)")
    args = ap.parse_args()
    parts = []
    parts.append(f"// gb_bitslice.cuh -- GENERATED by tools/gen_bitslice.py --code {args.code}; do not edit.")
    parts.append("//")
    parts.append("// Bit-sliced ascending candidate scan of the fused check (K3): one lane,")
    parts.append("// 32 consecutive evens, odd prime candidates in ascending order, the minimal")
    parts.append("// p of each even recorded as a monotone code of p in bit planes.  Follows")
    parts.append("// phase1_verify's scan order (reference proj/src/verifier.cpp:66-88).")
    parts.append("#pragma once")
    parts.append("#include <cstdint>")
    parts.append("")
    parts.append("namespace gbk {")
    parts.append("")
    if args.fma_every:
        parts.append("// 2^k; in constant memory so the IMAD funnel below is not folded into SHF")
        parts.append("__constant__ uint32_t c_pow2[32] = {" + ", ".join(f"{1 << k}u" for k in range(32)) + "};")
        parts.append("// funnel shift right of (hi:lo) by sh (0 < sh < 32) on the FMA pipe")
        parts.append("__device__ __forceinline__ uint32_t fsr_fma(uint32_t lo, uint32_t hi, int sh) {")
        parts.append("    const uint32_t K = c_pow2[32 - sh];")
        parts.append("    return hi * K + __umulhi(lo, K);")
        parts.append("}")
        parts.append("")
    parts.append("// ---- wheel-6 layout (k_verify_ws): one scan per residue class of n mod 6")
    pr0 = args.pbs_r0 or args.pbs6
    pr24 = args.pbs_r24 or args.pbs6
    pmax = max(pr0, pr24)
    npl = max(max(class_code(r, p, args.code) for p in odd_primes(pm) if p > 3 or r != 0)
              for r, pm in ((0, pr0), (2, pr24), (4, pr24))).bit_length()
    nw = scan6_words(pmax)
    parts.append(f"#define BS6_CODE {1 if args.code == 'c' else 0} // 1: planes hold the class code c, 0: z = (p - 3)/2")
    for r, pm in ((0, pr0), (2, pr24), (4, pr24)):
        code, n, _, _ = gen_scan6(f"bs6_scan_r{r}", r, pm, nplanes=npl, nw=nw, fma_every=args.fma_every,
                                  mode=args.code)
        parts.append("")
        parts.append(code)
    parts.append(f"constexpr uint32_t BS6_PMAX_R0 = {pr0};   // class 0 scans p <= BS6_PMAX_R0")
    parts.append(f"constexpr uint32_t BS6_PMAX_R24 = {pr24};  // classes 2, 4 scan p <= BS6_PMAX_R24")
    parts.append(f"constexpr uint32_t BS6_PMAX = {pmax};")
    parts.append(f"constexpr int BS6_PLANES = {npl};")
    parts.append(f"constexpr int BS6_WORDS = {nw};    // tile words per array a scan reads (WB-{nw - 1} .. WB)")
    parts.append(f"#define BS6_NWORDS {nw} // the same for the preprocessor (scan call sites)")
    parts.append("")
    parts.append("} // namespace gbk")
    with open(OUT, "w") as f:
        f.write("\n".join(parts) + "\n")
    print("wrote", OUT)


if __name__ == "__main__":
    main()
