"""CPU, world_size 2 over gloo: the N>1 path of bench.py / the multi-GPU
runner without GPUs -- two ranks steal segments from ONE shared cursor
(gb_pool over POSIX shared memory, claim_next semantics pool.cpp:24-31),
every segment is claimed exactly once, and one all-gather merges the
per-rank records with run_workers' rules (pool.cpp:159-174)."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, shm, start, limit, seg, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2603_07850_b200 as gb
    from paper_2603_07850_b200 import dist as gd
    pool = None
    if rank == 0:
        pool = gb.Pool(start, limit, seg, shm_name=shm, create=True)
    dist.barrier()
    if rank != 0:
        pool = gb.Pool(start, limit, seg, shm_name=shm, create=False)
    claimed = []
    # interleave claims so both ranks really compete for the cursor
    while (j := pool.claim()) is not None:
        claimed.append(j)
    # a fake per-rank "result": each claimed segment contributes its evens,
    # p = index+3 at n = a (a synthetic MinPrimeMax stream), hash of a
    res = dict(evens=0, unverified=0, phase2=0, sum_pmin=0, pos_hash=0, max_p=0, max_n=0,
               segments=0, n_ce=0, ce=[])
    for a, b, i in claimed:
        res["evens"] += (b - a) // 2 + 1
        res["segments"] += 1
        res["sum_pmin"] = (res["sum_pmin"] + (i % 7) + 3) % (1 << 64)
        res["pos_hash"] = (res["pos_hash"] + a * 0x9E3779B97F4A7C15) % (1 << 64)
        p = (i % 7) + 3
        if p > res["max_p"] or (p == res["max_p"] and a < res["max_n"]):
            res["max_p"], res["max_n"] = p, a
    merged = gd.allgather_merge(res)
    dist.barrier()
    pool.close(unlink=(rank == 0))
    q.put((rank, claimed, merged))
    dist.destroy_process_group()


@pytest.mark.parametrize("start,limit,seg", [(4, 2_000_002, 1000), ((1 << 64) - 200_002, (1 << 64) - 2, 997)])
def test_two_ranks_share_one_cursor_and_merge(start, limit, seg):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    shm = f"/gb_gloo_{os.getpid()}_{port}"
    procs = [ctx.Process(target=_worker, args=(r, 2, port, shm, start, limit, seg, q)) for r in (0, 1)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    claimed = sorted(j for _, c, _ in out for j in c)
    span = 2 * seg
    n_seg = (limit - start) // span + 1
    assert [j[2] for j in claimed] == list(range(n_seg))        # exactly once
    assert claimed[0][0] == start and claimed[-1][1] == limit
    assert all(b2 + 2 == a2 for (_, b2, _), (a2, _, _) in zip(claimed, claimed[1:]))
    m0, m1 = out[0][2], out[1][2]
    assert m0 == m1                                              # same on every rank
    assert m0["evens"] == (limit - start) // 2 + 1 and m0["segments"] == n_seg
    want_max = max(range(n_seg), key=lambda i: ((i % 7) + 3, -i))
    assert m0["max_p"] == (want_max % 7) + 3 and m0["max_n"] == start + want_max * span


def test_merge_rules():
    from paper_2603_07850_b200 import dist as gd
    a = dict(evens=5, unverified=1, phase2=1, sum_pmin=(1 << 64) - 1, pos_hash=3, max_p=7,
             max_n=100, segments=1, n_ce=1, ce=[50])
    b = dict(evens=6, unverified=0, phase2=0, sum_pmin=2, pos_hash=4, max_p=7, max_n=90,
             segments=2, n_ce=1, ce=[20])
    c = dict(evens=0, unverified=0, phase2=0, sum_pmin=0, pos_hash=0, max_p=0, max_n=0,
             segments=0, n_ce=0, ce=[])
    m = gd.merge([a, b, c])
    assert m["sum_pmin"] == 1 and m["evens"] == 11 and (m["max_p"], m["max_n"]) == (7, 90)
    assert m["ce"] == [20, 50] and m["n_ce"] == 2
    assert gd.unpack(gd.pack(m)) == m


def _stop_worker(rank, world, port, shm, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2603_07850_b200 as gb
    start, limit, seg = 4, 2_000_002, 1000
    pool = gb.Pool(start, limit, seg, shm_name=shm, create=True) if rank == 0 else None
    dist.barrier()
    if rank != 0:
        pool = gb.Pool(start, limit, seg, shm_name=shm, create=False)
    claimed = []
    if rank == 1:
        # rank 1 "finds a counterexample" in its second segment and stops
        # the shared pool, as run_workers / gb_drain_pool do (pool.cpp:104-111)
        claimed += [pool.claim(), pool.claim()]
        pool.request_stop()
    dist.barrier()
    stopped = pool.stop_requested
    while (j := pool.claim()) is not None:
        claimed.append(j)
    dist.barrier()
    pool.close(unlink=(rank == 0))
    q.put((rank, stopped, claimed))
    dist.destroy_process_group()


def test_stop_reaches_every_rank_on_a_shared_cursor():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    shm = f"/gb_gloo_stop_{os.getpid()}_{port}"
    procs = [ctx.Process(target=_stop_worker, args=(r, 2, port, shm, q)) for r in (0, 1)]
    for p in procs:
        p.start()
    out = dict((r, (s, c)) for r, s, c in (q.get(timeout=120) for _ in procs))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert out[0][0] and out[1][0]                 # both ranks see the stop word
    assert out[0][1] == []                         # rank 0 claims nothing after it
    assert [j[2] for j in out[1][1]] == [0, 1]     # only the segments claimed before the stop
