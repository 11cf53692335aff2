"""Internal paths the regular parity cases do not reach, each checked
against the oracle or against the regular path:

* straggler-list overflow (more than 2^20 evens of a batch need K4): the
  host re-runs the piece in sub-pieces that cannot overflow;
* pieces of 2^30 evens (MAX_SEG_EVENS) with user segments above it;
* run_workers with k in {1, 2, 4} GPU workers on one GPU (acceptance c6,
  acceptance.cpp:188-248) and the cooperative stop on a counterexample
  (pool.cpp:104-111) across two processes sharing one cursor."""
import multiprocessing as mp
import os
import socket

import pytest

pytestmark = pytest.mark.gpu


def test_straggler_overflow_rerun_matches_oracle(gpu):
    """p_small = 3: Phase 1 tries p = 3 only, so ~9 in 10 evens go to K4 and
    a 3 M-even segment overflows the 2^20-entry list."""
    import oracle
    a, b = 4, 6_000_002
    with gpu.Device(b, p_small=3) as dev:
        got = dev.verify_segment(a, b)
    # the oracle over 16 threads (same evens, totals are order-independent)
    want, _ = oracle.verify_range(a, b, 50_000, cover=b, p_small=3, threads=16)
    g, w = got.as_dict(), want.as_dict()
    for k in ("evens", "unverified", "phase2", "sum_pmin", "pos_hash", "max_p", "max_n", "n_ce"):
        assert g[k] == w[k], (k, g, w)
    assert g["unverified"] > (1 << 20)


def test_pieces_above_2_30_evens(gpu):
    """A 2^31-even user segment runs as two 2^30-even pieces; the merged
    record equals the same evens verified as ordinary 2e8 segments."""
    start, limit = 10**12, 10**12 + 2 * ((1 << 31) - 1)
    with gpu.Device(limit, max_seg_evens=1 << 31) as dev:
        big = dev.verify_segment(start, limit).as_dict()
    with gpu.Device(limit) as dev:
        pool = gpu.Pool(start, limit, 200_000_000)
        small = gpu.drain_pool(dev, pool).as_dict()
    assert big["evens"] == (1 << 31) == small["evens"]
    for k in ("unverified", "sum_pmin", "pos_hash", "max_p", "max_n"):
        assert big[k] == small[k], (k, big, small)


@pytest.mark.parametrize("k", [2, 4])
def test_run_range_worker_count_invariance(gpu, k):
    """acceptance c6: run_workers with k GPU workers round-robined on GPU 0
    gives the same totals as one worker; every worker claims segments."""
    r1, per1 = gpu.run_range(4, 10**11, devices=[0], workers=1)
    rk, perk = gpu.run_range(4, 10**11, devices=[0], workers=k)
    d1, dk = r1.as_dict(), rk.as_dict()
    for key in ("evens", "unverified", "phase2", "sum_pmin", "pos_hash", "max_p", "max_n", "segments"):
        assert d1[key] == dk[key], (key, d1, dk)
    assert len(perk) == k and sum(perk) == dk["segments"] == 250
    assert all(s > 0 for s in perk), perk


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _drain_rank(rank, world, port, shm, limit, inject, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2603_07850_b200 as gb
    pool = None
    if rank == 0:
        pool = gb.Pool(4, limit, 200_000_000, shm_name=shm, create=True)
    dist.barrier()
    if rank != 0:
        pool = gb.Pool(4, limit, 200_000_000, shm_name=shm, create=False)
    with gb.Device(limit, inject_fail=inject) as dev:
        r = gb.drain_pool(dev, pool).as_dict()
    stopped = pool.stop_requested
    dist.barrier()
    pool.close(unlink=(rank == 0))
    q.put((rank, r, stopped))
    dist.destroy_process_group()


def test_counterexample_stops_every_rank():
    """Two processes (gloo, both on GPU 0) drain one shared cursor with the
    same inject_fail: the rank that claims the segment holding it reports the
    counterexample and sets the pool's stop word, so neither rank drains the
    rest of the range (pool.cpp:104-111 across processes)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    shm = f"/gb_gpu_stop_{os.getpid()}_{port}"
    limit = 10**12  # 2,500 segments: far more than two ranks claim before the stop
    inject = 100_000_000  # in segment 0
    procs = [ctx.Process(target=_drain_rank, args=(r, 2, port, shm, limit, inject, q)) for r in (0, 1)]
    for p in procs:
        p.start()
    out = {}
    for _ in procs:
        rank, r, stopped = q.get(timeout=300)
        out[rank] = (r, stopped)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert out[0][1] and out[1][1]                       # both see the stop word
    assert out[0][0]["n_ce"] + out[1][0]["n_ce"] == 1     # one rank found it
    found = out[0][0] if out[0][0]["n_ce"] else out[1][0]
    assert found["ce"] == [inject]
    assert out[0][0]["segments"] + out[1][0]["segments"] < 100
