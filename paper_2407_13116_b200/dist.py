"""Multi-GPU plumbing for the study path: one process per GPU, contiguous index
shards, and ONE small all-reduce that combines the per-rank ErrorStats
(SURVEY.md §8e).

The payload is int64 slots so that a MAX all-reduce both reduces and
gathers:
  slots 0..4   the bit patterns of reG, reS1, reS2, reU, reV (non-negative
               doubles: their bit patterns order like the values; never -0/NaN
               on the absorbed path, oracle.hpp:251-263)
  slot 5       kappa_inf (MAX = OR)
  slot 6       2^62 - fail_key (MAX = the lowest failing key), -1 if none
  then one block per rank: kappa e, hi, lo, first index and the 19 branch
  counters, each 64-bit field split into two non-negative 32-bit halves; a
  rank writes only its own block and zeros elsewhere, so MAX is a gather.
The host merges the rank blocks in rank order with kog_stats_merge
(ErrorStats::merge, harness.hpp:96-105) — identical stats for any world size.
"""
from __future__ import annotations

import ctypes as C
import struct

import numpy as np

from . import capi

_FIELDS_PER_RANK = 4 + 19  # kappa e, hi, lo, index + 19 counters
HEAD = 7
NO_FAIL = -1
FAIL_BASE = 1 << 62


def shard(count: int, rank: int, world: int) -> tuple[int, int]:
    """[lo, hi) of rank's contiguous index range (last shard takes the remainder)."""
    per = count // world
    lo = rank * per
    hi = count if rank == world - 1 else lo + per
    return lo, hi


def _u64(x: float) -> int:
    return struct.unpack("<Q", struct.pack("<d", x))[0]


def _f64(u: int) -> float:
    return struct.unpack("<d", struct.pack("<Q", u & 0xFFFFFFFFFFFFFFFF))[0]


def _rank_fields(st: capi.kog_stats) -> list[int]:
    f = [st.max_kappa2.e & 0xFFFFFFFFFFFFFFFF, _u64(st.max_kappa2.hi), _u64(st.max_kappa2.lo), st.max_kappa2_index]
    f += list(st.t2p) + list(st.path)
    f += [st.tanpsi_inf, st.diag_swap, st.compose_minus, st.sigma_swap, st.prescale_inexact]
    return f


def pack(st: capi.kog_stats, rank: int, world: int) -> np.ndarray:
    buf = np.zeros(HEAD + 2 * _FIELDS_PER_RANK * world, dtype=np.int64)
    for k, name in enumerate(("reG", "reS1", "reS2", "reU", "reV")):
        buf[k] = _u64(getattr(st, name))
    buf[5] = 1 if st.kappa_inf else 0
    buf[6] = NO_FAIL if st.fail_key == 0xFFFFFFFFFFFFFFFF else FAIL_BASE - st.fail_key
    base = HEAD + 2 * _FIELDS_PER_RANK * rank
    for k, v in enumerate(_rank_fields(st)):
        buf[base + 2 * k] = v >> 32
        buf[base + 2 * k + 1] = v & 0xFFFFFFFF
    return buf


def unpack(buf: np.ndarray, world: int) -> capi.kog_stats:
    lib = capi.load()
    total = capi.kog_stats()
    lib.kog_stats_init(C.byref(total))
    for r in range(world):
        base = HEAD + 2 * _FIELDS_PER_RANK * r
        v = [(int(buf[base + 2 * k]) << 32) | int(buf[base + 2 * k + 1]) for k in range(_FIELDS_PER_RANK)]
        part = capi.kog_stats()
        lib.kog_stats_init(C.byref(part))
        e = v[0] - (1 << 64) if v[0] >= (1 << 63) else v[0]
        part.max_kappa2 = capi.kog_extfloat(e, _f64(v[1]), _f64(v[2]))
        part.max_kappa2_index = v[3]
        for k in range(7):
            part.t2p[k] = v[4 + k]
            part.path[k] = v[11 + k]
        (part.tanpsi_inf, part.diag_swap, part.compose_minus, part.sigma_swap,
         part.prescale_inexact) = v[18:23]
        lib.kog_stats_merge(C.byref(total), C.byref(part))
    for k, name in enumerate(("reG", "reS1", "reS2", "reU", "reV")):
        setattr(total, name, _f64(int(buf[k])))
    total.kappa_inf = int(buf[5])
    total.fail_key = 0xFFFFFFFFFFFFFFFF if int(buf[6]) == NO_FAIL else FAIL_BASE - int(buf[6])
    return total


def allreduce_stats(st: capi.kog_stats, group=None, device=None) -> capi.kog_stats:
    """Combine per-rank stats with one MAX all-reduce (NCCL on `device`, or
    gloo on CPU when device is None)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    t = torch.from_numpy(pack(st, rank, world))
    if device is not None:
        t = t.to(device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return unpack(t.cpu().numpy(), world)
