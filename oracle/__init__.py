"""ctypes bindings for the CPU oracle (oracle/liboracle.so) and the compiled
reference (oracle/_ref/libref.so, oracle/_ref/goldbach_ref).

TEST INFRASTRUCTURE ONLY: the product package paper_2603_07850_b200 never
imports this module.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs use it, always as the checker or the
timed CPU baseline, never as the thing measured for the GPU path.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_DIR = os.path.join(HERE, "_ref")
REF_LIB_PATH = os.path.join(REF_DIR, "libref.so")
REF_BIN = os.path.join(REF_DIR, "goldbach_ref")

GB_REC_MAX_CE = 16


class SegRecord(C.Structure):
    """Mirror of gb_seg_record (include/goldbach_b200.h)."""

    _fields_ = [
        ("a", C.c_uint64), ("b", C.c_uint64),
        ("evens_checked", C.c_uint64), ("unverified_p1", C.c_uint64),
        ("phase2_resolved", C.c_uint64), ("pmin_sum", C.c_uint64),
        ("pmin_hash", C.c_uint64), ("max_p", C.c_uint64), ("max_n", C.c_uint64),
        ("n_counterexamples", C.c_uint64),
        ("counterexamples", C.c_uint64 * GB_REC_MAX_CE),
        ("elapsed_seconds", C.c_double),
    ]

    def key(self) -> tuple:
        """Everything that must be bit-exact (elapsed time excluded)."""
        nce = min(self.n_counterexamples, GB_REC_MAX_CE)
        return (self.a, self.b, self.evens_checked, self.unverified_p1,
                self.phase2_resolved, self.pmin_sum, self.pmin_hash,
                self.max_p, self.max_n, self.n_counterexamples,
                tuple(self.counterexamples[i] for i in range(nce)))

    def as_dict(self) -> dict:
        k = self.key()
        names = ["a", "b", "evens", "unverified", "phase2", "sum_pmin",
                 "pos_hash", "max_p", "max_n", "n_ce", "ce"]
        d = dict(zip(names, k))
        d["ce"] = list(d["ce"])
        return d


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FileNotFoundError(f"{LIB_PATH} missing: run `make -C oracle`")
        L = C.CDLL(LIB_PATH)
        u64, i64, p64 = C.c_uint64, C.c_int64, C.POINTER(C.c_uint64)
        L.or_is_prime_u64.argtypes = [u64]; L.or_is_prime_u64.restype = C.c_int
        L.or_modpow.argtypes = [u64, u64, u64]; L.or_modpow.restype = u64
        L.or_modmul.argtypes = [u64, u64, u64]; L.or_modmul.restype = u64
        L.or_simple_sieve.argtypes = [u64, p64, u64]; L.or_simple_sieve.restype = i64
        L.or_sqrt_bound.argtypes = [u64]; L.or_sqrt_bound.restype = u64
        L.or_build_base_primes.argtypes = [u64, C.POINTER(C.c_uint32), u64, p64]
        L.or_build_base_primes.restype = i64
        L.or_first_tile_index.argtypes = [u64, u64, u64, p64]; L.or_first_tile_index.restype = C.c_int
        L.or_tiled_sieve_segment.argtypes = [u64, u64, C.POINTER(C.c_uint32), u64, u64, u64, p64]
        L.or_tiled_sieve_segment.restype = C.c_int
        L.or_sieve_range_for.argtypes = [u64, u64, u64, p64, p64]; L.or_sieve_range_for.restype = C.c_int
        L.or_phase1_pmin.argtypes = [u64, u64, p64, u64, p64, u64, u64, p64]
        L.or_phase1_pmin.restype = C.c_int
        L.or_phase2_resolve.argtypes = [u64, u64]; L.or_phase2_resolve.restype = u64
        L.or_verify_segment.argtypes = [u64, u64, u64, u64, u64, C.POINTER(SegRecord)]
        L.or_verify_segment.restype = C.c_int
        L.or_verify_range.argtypes = [u64, u64, u64, u64, u64, C.c_int, C.POINTER(SegRecord), p64]
        L.or_verify_range.restype = C.c_int
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_LIB_PATH)


def ref():
    global _ref
    if _ref is None:
        if not ref_available():
            raise FileNotFoundError(f"{REF_LIB_PATH} missing: run oracle/build_ref.sh")
        L = C.CDLL(REF_LIB_PATH)
        u64, p64 = C.c_uint64, C.POINTER(C.c_uint64)
        L.ref_is_prime.argtypes = [u64]; L.ref_is_prime.restype = C.c_int
        L.ref_base_primes.argtypes = [u64, C.POINTER(C.c_uint32), u64, p64]
        L.ref_base_primes.restype = C.c_int64
        L.ref_sieve.argtypes = [u64, u64, u64, u64, p64]; L.ref_sieve.restype = C.c_int
        L.ref_phase1_pmin.argtypes = [u64, u64, u64, u64, p64]; L.ref_phase1_pmin.restype = C.c_int
        L.ref_phase2_resolve.argtypes = [u64, u64, p64]; L.ref_phase2_resolve.restype = C.c_int
        L.ref_segment_record.argtypes = [u64, u64, u64, u64, u64, C.POINTER(SegRecord)]
        L.ref_segment_record.restype = C.c_int
        L.ref_segment_record1.argtypes = [u64, u64, u64, u64, u64, C.POINTER(SegRecord)]
        L.ref_segment_record1.restype = C.c_int
        _ref = L
    return _ref


# ---------------------------------------------------------------- oracle API
def is_prime(n: int) -> bool:
    return bool(lib().or_is_prime_u64(n))


def sqrt_bound(cover: int) -> int:
    return lib().or_sqrt_bound(cover)


def base_primes(cover: int):
    import numpy as np
    s = C.c_uint64()
    n = lib().or_build_base_primes(cover, None, 0, C.byref(s))
    out = np.zeros(max(n, 1), dtype=np.uint32)
    lib().or_build_base_primes(cover, out.ctypes.data_as(C.POINTER(C.c_uint32)), n, C.byref(s))
    return s.value, out[:n]


def simple_sieve(limit: int):
    import numpy as np
    n = lib().or_simple_sieve(limit, None, 0)
    out = np.zeros(n, dtype=np.uint64)
    lib().or_simple_sieve(limit, out.ctypes.data_as(C.POINTER(C.c_uint64)), n)
    return out


def first_tile_index(p: int, tile_lo: int, seg_hi: int):
    idx = C.c_uint64()
    rc = lib().or_first_tile_index(p, tile_lo, seg_hi, C.byref(idx))
    if rc < 0:
        raise ValueError("ParamError")
    return idx.value if rc == 1 else None


def sieve_words(lo: int, hi: int, cover: int | None = None, odds_per_tile: int = 32768):
    """OddBitset words of tiled_sieve_segment(lo, hi, build_base_primes(cover))."""
    import numpy as np
    s, base = base_primes(cover if cover is not None else hi)
    n_bits = (hi - lo) // 2 + 1
    words = np.zeros((n_bits + 63) // 64 + 1, dtype=np.uint64)
    rc = lib().or_tiled_sieve_segment(lo, hi, base.ctypes.data_as(C.POINTER(C.c_uint32)),
                                      len(base), s, odds_per_tile,
                                      words.ctypes.data_as(C.POINTER(C.c_uint64)))
    if rc:
        raise ValueError("ParamError")
    return words[: (n_bits + 63) // 64]


def sieve_range_for(a: int, b: int, p_small: int):
    lo, hi = C.c_uint64(), C.c_uint64()
    if lib().or_sieve_range_for(a, b, p_small, C.byref(lo), C.byref(hi)):
        raise ValueError("ParamError")
    return lo.value, hi.value


def phase1_pmin(a: int, b: int, p_small: int = 1_000_000, cover: int | None = None):
    """p_min per even of [a, b] (0 = not certified by Phase 1)."""
    import numpy as np
    lo, hi = sieve_range_for(a, b, p_small)
    words = sieve_words(lo, hi, cover if cover is not None else b)
    small = simple_sieve(p_small)[1:].copy()
    n = (b - a) // 2 + 1
    out = np.zeros(n, dtype=np.uint64)
    rc = lib().or_phase1_pmin(a, b, small.ctypes.data_as(C.POINTER(C.c_uint64)), len(small),
                              words.ctypes.data_as(C.POINTER(C.c_uint64)), lo, hi,
                              out.ctypes.data_as(C.POINTER(C.c_uint64)))
    if rc:
        raise ValueError(f"phase1 rc={rc}")
    return out


def phase2_resolve(n: int, p_small: int) -> int:
    return lib().or_phase2_resolve(n, p_small)


def verify_segment(a: int, b: int, cover: int | None = None, p_small: int = 1_000_000,
                   inject_fail: int = 0) -> SegRecord:
    rec = SegRecord()
    rc = lib().or_verify_segment(a, b, cover if cover is not None else b, p_small,
                                 inject_fail, C.byref(rec))
    if rc:
        raise ValueError(f"or_verify_segment rc={rc}")
    return rec


def verify_range(start: int, limit: int, seg_size: int = 200_000_000,
                 cover: int | None = None, p_small: int = 1_000_000, threads: int = 1):
    rec = SegRecord()
    segs = C.c_uint64()
    rc = lib().or_verify_range(start, limit, seg_size, cover if cover is not None else limit,
                               p_small, threads, C.byref(rec), C.byref(segs))
    if rc:
        raise ValueError(f"or_verify_range rc={rc}")
    return rec, segs.value


# ------------------------------------------------------- compiled reference
def ref_segment_record(a: int, b: int, cover: int | None = None, p_small: int = 1_000_000,
                       inject_fail: int = 0) -> SegRecord:
    rec = SegRecord()
    rc = ref().ref_segment_record(a, b, cover if cover is not None else b, p_small,
                                  inject_fail, C.byref(rec))
    if rc:
        raise ValueError(f"ref_segment_record rc={rc}")
    return rec


def ref_segment_record1(a: int, b: int, cover: int | None = None, p_small: int = 1_000_000,
                        inject_fail: int = 0) -> SegRecord:
    """Single-pass reference record (same reference functions, same order as
    verify_segment; see oracle/ref_shim.cpp ref_segment_record1)."""
    rec = SegRecord()
    rc = ref().ref_segment_record1(a, b, cover if cover is not None else b, p_small,
                                   inject_fail, C.byref(rec))
    if rc:
        raise ValueError(f"ref_segment_record1 rc={rc}")
    return rec


def ref_phase1_pmin(a: int, b: int, p_small: int = 1_000_000, cover: int | None = None):
    import numpy as np
    out = np.zeros((b - a) // 2 + 1, dtype=np.uint64)
    rc = ref().ref_phase1_pmin(a, b, cover if cover is not None else b, p_small,
                               out.ctypes.data_as(C.POINTER(C.c_uint64)))
    if rc:
        raise ValueError("ref_phase1_pmin failed")
    return out


def ref_sieve_words(lo: int, hi: int, cover: int | None = None, tile: int = 32768):
    import numpy as np
    n = (hi - lo) // 2 + 1
    words = np.zeros((n + 63) // 64, dtype=np.uint64)
    if ref().ref_sieve(lo, hi, cover if cover is not None else hi, tile,
                       words.ctypes.data_as(C.POINTER(C.c_uint64))):
        raise ValueError("ref_sieve failed")
    return words
