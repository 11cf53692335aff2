"""B200-native Goldbach verifier (drop-in for the verification path of
arXiv 2603.07850, "GoldbachGPU v2.0").

The product is the native library ``libgoldbach_b200.so`` built from
``csrc/`` (sm_100a CUDA kernels + the C-ABI of ``include/goldbach_b200.h`` +
the C++ host layer mirroring ``proj/include/goldbach``).  This module is a
thin ctypes binding for tests and ``bench.py``; it never computes anything
itself and never falls back to a CPU path -- importing it without the built
library raises.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

__all__ = [
    "LIB_PATH", "GB_REC_MAX_CE", "SegRecord", "RunResult", "GoldbachError", "ParamError",
    "ResourceError", "InternalError", "DeviceError", "Device", "Pool", "device_count",
    "lib", "run_range", "drain_pool", "version",
]

HERE = os.path.dirname(os.path.abspath(__file__))
DEFAULT_LIB_PATH = os.path.join(HERE, "libgoldbach_b200.so")
# Tools-only switch: tools/variants.sh timing runs load a differently built
# copy with GB_LIB_PATH, honoured only together with GB_TOOLS_LIB_OVERRIDE=1
# so a stray environment variable cannot swap the product library.
_override = os.environ.get("GB_LIB_PATH")
if _override and os.environ.get("GB_TOOLS_LIB_OVERRIDE") == "1":
    import sys as _sys
    print(f"paper_2603_07850_b200: tools override, loading {_override}", file=_sys.stderr)
    LIB_PATH = _override
else:
    LIB_PATH = DEFAULT_LIB_PATH
CLI_PATH = os.path.join(HERE, "bin", "goldbach")
GB_REC_MAX_CE = 16


class GoldbachError(RuntimeError):
    code = -1


class ParamError(GoldbachError, ValueError):        # errors.hpp:9-11
    code = 1


class ResourceError(GoldbachError):                 # errors.hpp:14-16
    code = 2


class InternalError(GoldbachError):                 # errors.hpp:20-22
    code = 3


class DeviceError(GoldbachError):
    code = 4


_ERRS = {1: ParamError, 2: ResourceError, 3: InternalError, 4: DeviceError}


class SegRecord(C.Structure):
    """gb_seg_record: SegmentReport (verifier.hpp:107-114) + checksum."""

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
        nce = min(self.n_counterexamples, GB_REC_MAX_CE)
        return (self.a, self.b, self.evens_checked, self.unverified_p1,
                self.phase2_resolved, self.pmin_sum, self.pmin_hash,
                self.max_p, self.max_n, self.n_counterexamples,
                tuple(self.counterexamples[i] for i in range(nce)))

    def as_dict(self) -> dict:
        names = ["a", "b", "evens", "unverified", "phase2", "sum_pmin",
                 "pos_hash", "max_p", "max_n", "n_ce", "ce"]
        d = dict(zip(names, self.key()))
        d["ce"] = list(d["ce"])
        return d


class Params(C.Structure):
    _fields_ = [("cover_limit", C.c_uint64), ("p_small", C.c_uint64),
                ("phase2_limit", C.c_uint64), ("batch_size", C.c_uint64),
                ("inject_fail", C.c_uint64), ("max_seg_evens", C.c_uint64)]


class RunResult(C.Structure):
    """gb_run_result: RunResult (pool.hpp:114-123) + checksum."""

    _fields_ = [
        ("evens_checked", C.c_uint64), ("unverified_total", C.c_uint64),
        ("phase2_total", C.c_uint64), ("pmin_sum", C.c_uint64), ("pmin_hash", C.c_uint64),
        ("max_p", C.c_uint64), ("max_n", C.c_uint64), ("segments", C.c_uint64),
        ("n_counterexamples", C.c_uint64), ("counterexamples", C.c_uint64 * GB_REC_MAX_CE),
        ("wall_seconds", C.c_double),
    ]

    def as_dict(self) -> dict:
        nce = min(self.n_counterexamples, GB_REC_MAX_CE)
        return dict(evens=self.evens_checked, unverified=self.unverified_total,
                    phase2=self.phase2_total, sum_pmin=self.pmin_sum, pos_hash=self.pmin_hash,
                    max_p=self.max_p, max_n=self.max_n, segments=self.segments,
                    n_ce=self.n_counterexamples,
                    ce=[self.counterexamples[i] for i in range(nce)],
                    wall_seconds=self.wall_seconds)


_lib = None


def lib():
    """Load the native library (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `make` or "
                          "`python -c 'import __graft_entry__ as g; g.build()'` -- there is no "
                          "CPU fallback")
    L = C.CDLL(LIB_PATH)
    u64, i32 = C.c_uint64, C.c_int
    p64 = C.POINTER(C.c_uint64)
    vp = C.c_void_p
    sig = {
        "gb_version": ([], C.c_char_p),
        "gb_device_count": ([C.POINTER(i32)], i32),
        "gb_open": ([i32, C.POINTER(Params), C.POINTER(vp)], i32),
        "gb_close": ([vp], i32),
        "gb_last_error": ([vp], C.c_char_p),
        "gb_set_inject_fail": ([vp, u64], i32),
        "gb_verify_segment": ([vp, u64, u64, C.POINTER(SegRecord)], i32),
        "gb_max_inflight": ([vp, C.POINTER(i32)], i32),
        "gb_submit_segment": ([vp, u64, u64, u64], i32),
        "gb_wait_segment": ([vp, C.POINTER(SegRecord), p64], i32),
        "gb_base_primes": ([vp, p64, p64, C.POINTER(C.c_uint32), u64], i32),
        "gb_sieve_interval": ([vp, u64, u64, p64, u64], i32),
        "gb_phase1_pmin": ([vp, u64, u64, p64, u64], i32),
        "gb_is_prime_batch": ([vp, p64, C.POINTER(C.c_uint8), u64], i32),
        "gb_phase2_resolve": ([vp, u64, p64], i32),
        "gb_launch_count": ([vp, p64], i32),
        "gb_kernel_times": ([vp, C.POINTER(C.c_double), p64, i32], i32),
        "gb_set_timing": ([vp, i32], i32),
        "gb_set_bucket": ([vp, i32], i32),
        "gb_debug_tile": ([vp, u64, u64, C.c_uint32, C.POINTER(C.c_uint32), u64, C.POINTER(C.c_uint32),
                           C.POINTER(C.c_int64)], i32),
        "gb_bucket_info": ([vp, p64], i32),
        "gb_io_bytes": ([vp, p64, p64], i32),
        "gb_flush_l2": ([vp], i32),
        "gb_synchronize": ([vp], i32),
        "gb_primes_upto": ([vp, u64, C.POINTER(C.c_uint32), u64, p64], i32),
        "gb_device_timer": ([vp, i32, C.POINTER(C.c_double)], i32),
        "gb_smem_peak": ([vp, C.POINTER(C.c_double)], i32),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _bind_pool(L)
    _lib = L
    return L


def _bind_pool(L):
    """Pool / run entry points (include/goldbach_b200_pool.h), if built."""
    u64, i32, vp = C.c_uint64, C.c_int, C.c_void_p
    p64 = C.POINTER(C.c_uint64)
    sig = {
        "gb_pool_create": ([u64, u64, u64, C.c_char_p, i32, C.POINTER(vp)], i32),
        "gb_pool_claim": ([vp, p64, p64, p64], i32),
        "gb_pool_destroy": ([vp, i32], i32),
        "gb_pool_request_stop": ([vp], i32),
        "gb_pool_stop_requested": ([vp], i32),
        "gb_drain_pool": ([vp, vp, i32, C.POINTER(RunResult)], i32),
        "gb_run_range": ([u64, u64, u64, u64, u64, C.POINTER(i32), i32, i32, i32,
                          C.POINTER(RunResult), p64], i32),
        "gb_estimate_device_bytes": ([u64, u64, u64], u64),
        "gb_device_memory": ([i32, p64, p64], i32),
        "gb_pool_last_error": ([], C.c_char_p),
        "gb_primes_upto": ([vp, u64, C.POINTER(C.c_uint32), u64, p64], i32),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name, None)
        if fn is not None:
            fn.argtypes = args
            fn.restype = res


def _check(rc: int, handle=None):
    if rc == 0:
        return
    msg = lib().gb_last_error(handle).decode(errors="replace")
    raise _ERRS.get(rc, GoldbachError)(msg)


def version() -> str:
    return lib().gb_version().decode()


def device_count() -> int:
    n = C.c_int()
    _check(lib().gb_device_count(C.byref(n)))
    return n.value


class Device:
    """One GPU with resident tables: the gb_dev handle (gb_open)."""

    def __init__(self, cover_limit: int, p_small: int = 1_000_000, device: int = 0,
                 inject_fail: int = 0, max_seg_evens: int = 200_000_000,
                 phase2_limit: int = 100_000_000, batch_size: int = 2_000_000):
        L = lib()
        prm = Params(cover_limit, p_small, phase2_limit, batch_size, inject_fail, max_seg_evens)
        h = C.c_void_p()
        rc = L.gb_open(device, C.byref(prm), C.byref(h))
        _check(rc, None)
        self._h = h
        self.cover_limit = cover_limit
        self.p_small = p_small
        self.device = device

    # -- lifecycle
    def close(self):
        if getattr(self, "_h", None):
            lib().gb_close(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    # -- the drop-in boundary
    def verify_segment(self, a: int, b: int) -> SegRecord:
        rec = SegRecord()
        _check(lib().gb_verify_segment(self._h, a, b, C.byref(rec)), self._h)
        return rec

    def submit(self, a: int, b: int, tag: int = 0):
        _check(lib().gb_submit_segment(self._h, a, b, tag), self._h)

    def wait(self):
        rec = SegRecord()
        tag = C.c_uint64()
        _check(lib().gb_wait_segment(self._h, C.byref(rec), C.byref(tag)), self._h)
        return rec, tag.value

    def max_inflight(self) -> int:
        d = C.c_int()
        _check(lib().gb_max_inflight(self._h, C.byref(d)), self._h)
        return d.value

    def set_inject_fail(self, n: int):
        _check(lib().gb_set_inject_fail(self._h, n), self._h)

    # -- parity hooks
    def base_primes(self, copy: bool = True):
        import numpy as np
        s, n = C.c_uint64(), C.c_uint64()
        _check(lib().gb_base_primes(self._h, C.byref(s), C.byref(n), None, 0), self._h)
        out = None
        if copy:
            out = np.zeros(max(n.value, 1), dtype=np.uint32)
            _check(lib().gb_base_primes(self._h, None, None,
                                        out.ctypes.data_as(C.POINTER(C.c_uint32)), n.value),
                   self._h)
            out = out[: n.value]
        return s.value, n.value, out

    def sieve_words(self, lo: int, hi: int):
        import numpy as np
        nw = ((hi - lo) // 2 + 64) // 64
        w = np.zeros(nw, dtype=np.uint64)
        _check(lib().gb_sieve_interval(self._h, lo, hi, w.ctypes.data_as(C.POINTER(C.c_uint64)),
                                       nw), self._h)
        return w

    def phase1_pmin(self, a: int, b: int):
        import numpy as np
        n = (b - a) // 2 + 1
        out = np.zeros(n, dtype=np.uint64)
        _check(lib().gb_phase1_pmin(self._h, a, b, out.ctypes.data_as(C.POINTER(C.c_uint64)), n),
               self._h)
        return out

    def is_prime(self, values: Sequence[int]):
        import numpy as np
        v = np.ascontiguousarray(np.asarray(values, dtype=np.uint64))
        out = np.zeros(len(v), dtype=np.uint8)
        _check(lib().gb_is_prime_batch(self._h, v.ctypes.data_as(C.POINTER(C.c_uint64)),
                                       out.ctypes.data_as(C.POINTER(C.c_uint8)), len(v)), self._h)
        return out.astype(bool)

    def phase2_resolve(self, n: int) -> int:
        p = C.c_uint64()
        _check(lib().gb_phase2_resolve(self._h, n, C.byref(p)), self._h)
        return p.value

    def launch_count(self) -> int:
        n = C.c_uint64()
        _check(lib().gb_launch_count(self._h, C.byref(n)), self._h)
        return n.value

    def set_timing(self, mode):
        """0/False off, 1/True event timing, 2 timing with serialised batches."""
        _check(lib().gb_set_timing(self._h, int(mode)), self._h)

    def tile_words(self) -> int:
        """Words per class array of the fused kernel's wheel-6 tile."""
        nw = C.c_uint32()
        _check(lib().gb_debug_tile(self._h, 0, 0, 0, None, 0, C.byref(nw), None), self._h)
        return nw.value

    def debug_tile(self, a: int, b: int, block: int):
        """The fused kernel's sieved wheel-6 tile of one block (parity hook):
        (origin Q, A words, B words); A bit k <-> q = Q + 6k, B bit k <->
        q = Q + 4 + 6k."""
        import numpy as np
        nw = C.c_uint32()
        q = C.c_int64()
        n = self.tile_words()
        w = np.zeros(2 * n, dtype=np.uint32)
        _check(lib().gb_debug_tile(self._h, a, b, block, w.ctypes.data_as(C.POINTER(C.c_uint32)), 2 * n,
                                   C.byref(nw), C.byref(q)), self._h)
        return q.value, w[:n], w[n:]

    def set_bucket(self, enabled: bool):
        """Mask fill of the large tile primes on/off (results are identical)."""
        _check(lib().gb_set_bucket(self._h, 1 if enabled else 0), self._h)

    def bucket_info(self) -> dict:
        v = (C.c_uint64 * 8)()
        _check(lib().gb_bucket_info(self._h, v), self._h)
        keys = ("active", "p0", "primes", "range_cells", "large_primes")
        return dict(zip(keys, list(v)))

    def io_bytes(self):
        h, d = C.c_uint64(), C.c_uint64()
        _check(lib().gb_io_bytes(self._h, C.byref(h), C.byref(d)), self._h)
        return h.value, d.value

    def flush_l2(self):
        _check(lib().gb_flush_l2(self._h), self._h)

    def synchronize(self):
        _check(lib().gb_synchronize(self._h), self._h)

    def primes_upto(self, limit: int):
        import numpy as np
        n = C.c_uint64()
        _check(lib().gb_primes_upto(self._h, limit, None, 0, C.byref(n)), self._h)
        out = np.zeros(max(n.value, 1), dtype=np.uint32)
        _check(lib().gb_primes_upto(self._h, limit, out.ctypes.data_as(C.POINTER(C.c_uint32)),
                                    n.value, C.byref(n)), self._h)
        return out[: n.value]

    def timer_start(self):
        """Drain the device and record the start event (gb_device_timer)."""
        _check(lib().gb_device_timer(self._h, 0, None), self._h)

    def timer_stop(self) -> float:
        """Drain the device, record the stop event; elapsed device ms."""
        ms = C.c_double()
        _check(lib().gb_device_timer(self._h, 1, C.byref(ms)), self._h)
        return ms.value

    def smem_peak(self) -> float:
        """Measured shared-memory load bandwidth, bytes/s."""
        v = C.c_double()
        _check(lib().gb_smem_peak(self._h, C.byref(v)), self._h)
        return v.value

    def kernel_times(self, reset: bool = False):
        ms = (C.c_double * 4)()
        nl = (C.c_uint64 * 4)()
        _check(lib().gb_kernel_times(self._h, ms, nl, 1 if reset else 0), self._h)
        return list(ms), list(nl)


class Pool:
    """WorkPool (pool.hpp:21-42); with shm_name the cursor lives in POSIX
    shared memory so every process on the node steals from one counter."""

    def __init__(self, start: int, limit: int, seg_size: int, shm_name: Optional[str] = None,
                 create: bool = True):
        h = C.c_void_p()
        name = shm_name.encode() if shm_name else None
        rc = lib().gb_pool_create(start, limit, seg_size, name, 1 if create else 0, C.byref(h))
        if rc:
            raise _ERRS.get(rc, GoldbachError)(lib().gb_pool_last_error().decode(errors="replace"))
        self._h = h
        self.shm_name = shm_name
        self.owner = create

    def claim(self):
        a, b, i = C.c_uint64(), C.c_uint64(), C.c_uint64()
        rc = lib().gb_pool_claim(self._h, C.byref(a), C.byref(b), C.byref(i))
        if rc < 0:
            raise _ERRS.get(-rc, GoldbachError)("gb_pool_claim failed")
        return (a.value, b.value, i.value) if rc == 1 else None

    def request_stop(self):
        """Cooperative stop (pool.cpp:104-111): later claims on this pool,
        in every process attached to the shared cursor, return None."""
        _check_pool(lib().gb_pool_request_stop(self._h))

    @property
    def stop_requested(self) -> bool:
        return bool(lib().gb_pool_stop_requested(self._h))

    def close(self, unlink: Optional[bool] = None):
        if getattr(self, "_h", None):
            lib().gb_pool_destroy(self._h, 1 if (self.owner if unlink is None else unlink) else 0)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h


def _check_pool(rc: int):
    if rc:
        raise _ERRS.get(rc, GoldbachError)(lib().gb_pool_last_error().decode(errors="replace"))


def estimate_device_bytes(cover_limit: int, p_small: int = 1_000_000,
                          max_seg_evens: int = 200_000_000) -> int:
    return lib().gb_estimate_device_bytes(cover_limit, p_small, max_seg_evens)


def drain_pool(dev: Device, pool: Pool, max_inflight: int = 0) -> RunResult:
    """One GPU worker's loop (pool.cpp:90-120) until the pool is exhausted."""
    res = RunResult()
    _check(lib().gb_drain_pool(dev.handle, pool.handle, max_inflight, C.byref(res)), dev.handle)
    return res


def run_range(start: int, limit: int, seg_size: int = 200_000_000, p_small: int = 1_000_000,
              inject_fail: int = 0, devices: Sequence[int] = (0,), workers: Optional[int] = None,
              progress: bool = False):
    """run_workers (pool.cpp:70-175) over `workers` GPU workers mapped onto
    `devices` round-robin: returns (RunResult, per_worker_segments)."""
    devs = list(devices)
    k = workers if workers is not None else len(devs)
    # the worker count exactly as gb_run_range computes it (pool_capi.cpp),
    # so per_worker_segments is sized for every entry the C side writes
    k = k if k and k > 0 else max(1, len(devs))
    arr = (C.c_int * len(devs))(*devs)
    res = RunResult()
    per = (C.c_uint64 * k)()
    rc = lib().gb_run_range(start, limit, seg_size, p_small, inject_fail, arr, len(devs), k,
                            1 if progress else 0, C.byref(res), per)
    if rc:
        raise _ERRS.get(rc, GoldbachError)(lib().gb_pool_last_error().decode(errors="replace"))
    return res, list(per)[:k]
