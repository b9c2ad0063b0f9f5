"""Multi-GPU sharding of the hot path.

Two independent partitions, one process per GPU:
  * encode: rank g bundles the contiguous point slice [g N / G, (g+1) N / G)
    into its own pending memories; ONE collective, an all-reduce (sum) of the
    library's packed pending buffer (memories + counts, 16 Dp + 16 bytes at
    delta = 1) over NCCL, is Alg. 3's fusion of identically
    configured agents; every rank then commits;
  * decode + entropy: rank g owns grid rows [g R / G, (g+1) R / G) and decodes
    h halo rows on each side (clipped), so the window entropy needs no
    communication.  Results stay sharded.

The helpers below are pure host logic (tested on CPU with gloo, world 2) plus
the one all-reduce call.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def point_shard(n: int, rank: int, world: int):
    """Contiguous equal index range [lo, hi) of n points for `rank`."""
    return n * rank // world, n * (rank + 1) // world


def row_band(rows: int, rank: int, world: int):
    """Row band [r0, r1) of the full grid owned by `rank`."""
    return rows * rank // world, rows * (rank + 1) // world


def decoded_rows(rows: int, r0: int, r1: int, halo: int):
    """Rows the decode evaluates for band [r0, r1): the band plus halo, clipped."""
    return max(0, r0 - halo), min(rows, r1 + halo)


def allreduce_pending(buf: torch.Tensor, group=None):
    """Sum the packed pending buffer (memories, then the per-slot point counts as
    integer-valued doubles; vsaogm.h: vsaogm_pending) over all ranks, in place: ONE
    collective per batch (Alg. 3 fusion)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        if buf.is_cuda and dist.get_backend(group) == "gloo":
            # gloo (CPU tests, several ranks sharing one GPU): host round trip, same sum
            host = buf.cpu()
            dist.all_reduce(host, op=dist.ReduceOp.SUM, group=group)
            buf.copy_(host)
        else:
            dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)


def fuse_and_commit(mapper, group=None, timer=None):
    """Alg. 3 across ranks, then m += pending on every rank (multi-rank mode).

    `timer`, if given, is a pair of CUDA events recorded on the current stream around the
    collective (the bench's all-reduce latency)."""
    buf = mapper.pending_buffer()
    if timer is not None:
        timer[0].record()
    allreduce_pending(buf, group)
    if timer is not None:
        timer[1].record()
    mapper.commit()
