"""Island model: one colony per GPU, best-tour exchange
every X iterations.

The device path is ``Colony.island_init`` / ``Colony.island_exchange``: NCCL
inside libacs_b200.so (min-allreduce of ``L_gb << 16 | rank``, then a
sum-allreduce in which only the winner contributes its tour, then a device-
side strictly-better adoption) -- no host round trip.

``exchange_host`` is the same protocol over a ``torch.distributed`` process
group with host buffers (gloo or nccl); it runs the identical decision logic
and exists so the multi-rank host logic is testable on CPU-only machines
(world_size 2, gloo) and usable where NCCL peers are unavailable.
"""
from __future__ import annotations

import numpy as np


RANK_BITS = 16
NO_KEY = (1 << 63) - 1          # no tour yet: never wins, adopts nothing
MAX_LEN = (1 << (63 - RANK_BITS)) - 1


def exchange_key(best_len: int, rank: int) -> int:
    """min over ranks selects the best colony; ties go to the lowest rank.
    Same layout as the device path (k_island_pack): L_gb << 16 | rank, and
    the sentinel NO_KEY for a colony that has no tour yet."""
    if rank < 0 or rank >= (1 << RANK_BITS):
        raise ValueError("island rank must fit in 16 bits")
    best_len = int(best_len)
    if best_len < 0 or best_len > MAX_LEN:
        return NO_KEY
    return (best_len << RANK_BITS) | rank


def decode_key(key: int):
    """(winner rank, global best length); (None, None) for NO_KEY."""
    if key == NO_KEY:
        return None, None
    return key & ((1 << RANK_BITS) - 1), key >> RANK_BITS


def exchange_host(colony, dist, group=None) -> int:
    """One exchange over torch.distributed.  ``colony`` provides
    ``best() -> (order, len)`` and ``set_best(order, len)`` (strictly-better
    adoption is enforced by the callee, as acs_gpu_set_best does).
    Returns the global best length."""
    import torch
    rank = dist.get_rank(group)
    order, length = colony.best()
    key = torch.tensor([exchange_key(length, rank)], dtype=torch.int64)
    dist.all_reduce(key, op=dist.ReduceOp.MIN, group=group)
    winner, glen = decode_key(int(key.item()))
    if winner is None:  # no rank has a tour yet
        return length
    buf = torch.from_numpy(np.ascontiguousarray(order, np.int64)) if rank == winner \
        else torch.zeros(len(order), dtype=torch.int64)
    dist.broadcast(buf, src=dist.get_global_rank(group, winner) if group is not None else winner, group=group)
    if glen < length:
        colony.set_best(buf.numpy().astype(np.uint32), glen)
    return glen


def run_islands(colony, dist, iterations: int, exchange_every: int, device_path: bool = True):
    """Drive one island: iterate, exchanging every ``exchange_every`` iterations.
    Returns the per-iteration global-best trace of this colony."""
    trace = []
    done = 0
    while done < iterations:
        chunk = min(exchange_every, iterations - done)
        st = colony.iterate(chunk)
        trace.extend(st["global_best_len"].tolist())
        done += chunk
        if dist.get_world_size() > 1:
            if device_path:
                colony.island_exchange()
            else:
                exchange_host(colony, dist)
    return trace
