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

import numpy as np

from . import capi


def shard(count: int, rank: int, world: int) -> tuple[int, int]:
    """[lo, hi) of rank's contiguous index range (last shard takes the
    remainder): kog_study_shard."""
    lo, hi = C.c_uint64(), C.c_uint64()
    capi.load().kog_study_shard(count, rank, world, C.byref(lo), C.byref(hi))
    return lo.value, hi.value


def pack(st: capi.kog_stats, rank: int, world: int) -> np.ndarray:
    """kog_stats_pack: this rank's stats as the int64 slot vector."""
    lib = capi.load()
    buf = np.zeros(lib.kog_stats_slot_count(world), dtype=np.int64)
    capi.check(lib.kog_stats_pack(C.byref(st), rank, world, buf.ctypes.data))
    return buf


def unpack(buf: np.ndarray, world: int) -> capi.kog_stats:
    """kog_stats_unpack: the MAX-reduced slot vector back into stats, the rank
    blocks merged in rank order."""
    buf = np.ascontiguousarray(buf, dtype=np.int64)
    out = capi.kog_stats()
    capi.check(capi.load().kog_stats_unpack(buf.ctypes.data, world, C.byref(out)))
    return out


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


class NcclStats:
    """The NCCL all-reduce of the stats slots issued from the library's C++
    side (kog_study_allreduce) on a communicator of its own: rank 0's unique id
    travels through torch.distributed (plumbing only), every rank builds its
    communicator on its current CUDA device."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist

        lib = capi.load()
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        uid = (C.c_uint8 * 128)()
        if self.rank == 0:
            capi.check(lib.kog_nccl_unique_id(uid, 128))
        box = [bytes(uid)]
        dist.broadcast_object_list(box, src=0, group=group)
        C.memmove(uid, box[0], 128)
        self.comm = C.c_void_p()
        capi.check(lib.kog_nccl_comm_init(uid, self.world, self.rank, C.byref(self.comm)))
        self._stream = torch.cuda.current_stream().cuda_stream

    def allreduce(self, st: capi.kog_stats) -> capi.kog_stats:
        out = capi.kog_stats.from_buffer_copy(bytes(st))
        capi.check(capi.load().kog_study_allreduce(self.comm, self.rank, self.world, C.byref(out), self._stream))
        return out

    def close(self):
        if self.comm:
            capi.load().kog_nccl_comm_destroy(self.comm)
            self.comm = C.c_void_p()
