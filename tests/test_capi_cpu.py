"""CPU: the C-ABI library loads and exports every symbol include/*.h
declares; host-side entry points that need no GPU behave like the
reference (WorkPool claim semantics, parameter errors)."""
import ctypes as C
import os
import re
import subprocess

import pytest

from conftest import ROOT

import paper_2603_07850_b200 as gb


def declared_functions():
    names = []
    for h in ("goldbach_b200.h", "goldbach_b200_pool.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names += re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(gb_[a-z_0-9]+)\s*\(", src, re.M)
    return sorted(set(names))


def test_library_exports_every_declared_symbol():
    L = gb.lib()
    names = declared_functions()
    assert len(names) >= 30, names
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    # the library is the sm_100a build
    out = subprocess.run(["cuobjdump", "--list-elf", gb.LIB_PATH], capture_output=True, text=True)
    if out.returncode == 0:
        assert "sm_100a" in out.stdout


def test_version_and_no_device_error():
    assert "sm_100a" in gb.version()
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except Exception:
        pass
    assert gb.device_count() == 0
    with pytest.raises(gb.GoldbachError):
        gb.Device(10**8)


def test_pool_claim_sequence_matches_reference():
    # test_pool.cpp:15-51: claim sequence and the short final segment
    p = gb.Pool(4, 100, 10)
    jobs = []
    while (j := p.claim()) is not None:
        jobs.append(j)
    assert jobs == [(4, 22, 0), (24, 42, 1), (44, 62, 2), (64, 82, 3), (84, 100, 4)]
    assert p.claim() is None
    p.close()


def test_pool_no_wrap_near_2_64():
    # test_pool.cpp:84-97
    top = (1 << 64) - 2
    p = gb.Pool(top - 40, top, 10)
    jobs = []
    while (j := p.claim()) is not None:
        jobs.append(j)
        assert len(jobs) < 10
    assert jobs[-1][1] == top and jobs[0][0] == top - 40
    assert sum((b - a) // 2 + 1 for a, b, _ in jobs) == 21


@pytest.mark.parametrize("args", [(5, 100, 10), (4, 101, 10), (2, 100, 10), (100, 4, 10),
                                  (4, 100, 0), (4, 100, 1 << 32)])
def test_pool_rejects_bad_bounds(args):
    with pytest.raises(gb.ParamError):
        gb.Pool(*args)


def test_shared_pool_attach_validates():
    name = f"/gb_test_{os.getpid()}"
    p = gb.Pool(4, 1000, 10, shm_name=name, create=True)
    q = gb.Pool(4, 1000, 10, shm_name=name, create=False)
    with pytest.raises(gb.ParamError):
        gb.Pool(4, 998, 10, shm_name=name, create=False)
    a = p.claim()
    b = q.claim()
    assert (a[2], b[2]) == (0, 1)  # one cursor
    q.close(unlink=False)
    p.close(unlink=True)


def test_device_bytes_estimate_scales():
    e12 = gb.estimate_device_bytes(10**12)
    e13 = gb.estimate_device_bytes(10**13)
    c5 = gb.estimate_device_bytes(4_000_000_100_000_000_000)
    assert 0 < e12 < e13 < c5
    assert c5 > 393_000_000  # 98.2 M base primes as u32
    assert c5 < 180 * 10**9


def test_cpp_host_unit_tests():
    exe = os.path.join(ROOT, "paper_2603_07850_b200", "bin", "test_host")
    if not os.path.exists(exe):
        pytest.skip("test_host not built")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    assert " 0 failed" in out.stdout


def test_reference_api_conformance_host():
    """Every symbol of the reference headers (proj/include/goldbach/*.hpp)
    with its exact signature compiles and links against this library
    (ref_api_conformance.cpp: static_asserts on pointer and member types);
    the host-only entry points return the reference tests' known answers."""
    exe = os.path.join(ROOT, "paper_2603_07850_b200", "bin", "ref_api_conformance")
    if not os.path.exists(exe):
        subprocess.run(["make", "-C", ROOT, "cli"], check=True, capture_output=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr[-2000:]
    assert "conformance ok" in out.stdout
