"""Multi-GPU plumbing of the verifier: one process per GPU, one shared
work-stealing cursor, one collective at the end.

Reference semantics followed:
  * claim_next        proj/src/pool.cpp:24-31 (the cursor lives in POSIX
                      shared memory, gb_pool_create, so every rank of the node
                      steals from ONE atomic counter -- no static partition)
  * run_workers merge proj/src/pool.cpp:159-174: evens / unverified / phase2 /
                      segments summed, MinPrimeMax merged (max p, smallest n
                      on ties, p = 0 ignored, verifier.hpp:53-66),
                      counterexamples concatenated and sorted.

The per-rank record is packed into a fixed-size u64 vector (signed int64
bit patterns, because torch has no uint64 collectives) and exchanged with a
single ``all_gather_into_tensor`` -- NCCL over NVLink on GPUs, gloo on CPU in
the tests.  Nothing here runs on the hot path.
"""
from __future__ import annotations

from typing import Iterable, List

GB_REC_MAX_CE = 16
MASK = (1 << 64) - 1
# evens, unverified, phase2, sum, hash, max_p, max_n, segments, n_ce, ce[16]
REC_LEN = 9 + GB_REC_MAX_CE


def _s64(x: int) -> int:
    x &= MASK
    return x - (1 << 64) if x >> 63 else x


def _u64(x: int) -> int:
    return int(x) & MASK


def pack(res: dict) -> List[int]:
    """dict (RunResult.as_dict() keys) -> REC_LEN signed 64-bit ints."""
    ce = list(res.get("ce", []))[:GB_REC_MAX_CE]
    v = [res["evens"], res["unverified"], res["phase2"], res["sum_pmin"], res["pos_hash"],
         res["max_p"], res["max_n"], res["segments"], res["n_ce"]]
    v += ce + [0] * (GB_REC_MAX_CE - len(ce))
    return [_s64(x) for x in v]


def unpack(v: Iterable[int]) -> dict:
    u = [_u64(x) for x in v]
    n_ce = u[8]
    return dict(evens=u[0], unverified=u[1], phase2=u[2], sum_pmin=u[3], pos_hash=u[4],
                max_p=u[5], max_n=u[6], segments=u[7], n_ce=n_ce,
                ce=u[9:9 + min(n_ce, GB_REC_MAX_CE)])


def merge(results: Iterable[dict]) -> dict:
    """run_workers' merge (pool.cpp:159-174) with MinPrimeMax::merge
    (verifier.hpp:60-65); sums wrap mod 2^64 like the u64 fields."""
    out = dict(evens=0, unverified=0, phase2=0, sum_pmin=0, pos_hash=0, max_p=0, max_n=0,
               segments=0, n_ce=0, ce=[])
    for r in results:
        for k in ("evens", "unverified", "phase2", "sum_pmin", "pos_hash", "segments", "n_ce"):
            out[k] = (out[k] + r[k]) & MASK
        p, n = r["max_p"], r["max_n"]
        if p != 0 and (p > out["max_p"] or (p == out["max_p"] and n < out["max_n"])):
            out["max_p"], out["max_n"] = p, n
        out["ce"] = sorted(out["ce"] + list(r["ce"]))[:GB_REC_MAX_CE]
    return out


def allgather_merge(res: dict, device=None, group=None) -> dict:
    """One all-gather of every rank's packed record, merged identically on
    every rank.  `device` is the tensor device of the backend (cuda:i for
    NCCL, cpu for gloo)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    mine = torch.tensor(pack(res), dtype=torch.int64, device=device)
    everyone = torch.empty(world * REC_LEN, dtype=torch.int64, device=device)
    dist.all_gather_into_tensor(everyone, mine, group=group)
    rows = everyone.view(world, REC_LEN).cpu().tolist()
    return merge(unpack(r) for r in rows)


def max_over_ranks(x: float, device=None, group=None) -> float:
    """Max of a per-rank float (step time) over all ranks."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def sum_over_ranks(x: int, device=None, group=None) -> int:
    import torch
    import torch.distributed as dist

    t = torch.tensor([int(x)], dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return int(t.item())
