"""Data parallelism over collocation points (BASELINE.json north_star (3)).

Every rank owns a contiguous, equal block of each point set (interior, boundary, initial),
evaluates its partial loss and gradient with the GLOBAL normalisers N_int and N_bi, and the flat
buffer [dL/dtheta | alpha*L_pde | L_bi | nonfinite | pad] is summed by ONE allreduce
(torch.distributed; NCCL over NVLink/NVSwitch on the B200 box).  Adam then runs replicated on
every rank on bit-identical inputs, so parameters stay identical without a broadcast.

The loss+grad evaluation is injected (`loss_grad_fn`) so that the host logic here is exercised
by world_size-2 gloo tests on CPU; in production it is HRKANNet.pinn_loss_grad.
"""
from __future__ import annotations

from typing import Callable, Optional, Sequence, Tuple


def shard_range(n: int, rank: int, world: int) -> Tuple[int, int]:
    """[lo, hi) of rank's contiguous block of n items (block sizes differ by at most one)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return (n * rank) // world, (n * (rank + 1)) // world


def shard(arr, rank: int, world: int):
    if arr is None:
        return None
    lo, hi = shard_range(len(arr), rank, world)
    return arr[lo:hi]


def dp_loss_grad(loss_grad_fn: Callable, sets: dict, rank: int, world: int, group=None,
                 allreduce: bool = True):
    """One data-parallel loss+grad evaluation.

    sets: {"interior", "forcing", "boundary", "g_boundary", "initial", "g_initial"} (full sets;
    each rank slices its shard here).  loss_grad_fn(interior=, forcing=, boundary=, g_boundary=,
    initial=, g_initial=, n_int_global=, n_bi_global=) -> flat buffer (torch tensor).
    Returns the allreduced buffer (identical on every rank)."""
    import torch.distributed as dist
    n_int = len(sets["interior"])
    n_bi = len(sets["boundary"]) + (0 if sets.get("initial") is None else len(sets["initial"]))
    local = {k: shard(v, rank, world) for k, v in sets.items()}
    out = loss_grad_fn(n_int_global=n_int, n_bi_global=n_bi, **local)
    if allreduce and world > 1:
        dist.all_reduce(out, op=dist.ReduceOp.SUM, group=group)
    return out
