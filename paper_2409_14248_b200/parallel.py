"""Data parallelism over collocation points (BASELINE.json north_star (3)).

Every rank owns a contiguous, equal block of each point set (interior, boundary, initial),
evaluates its partial loss and gradient with the GLOBAL normalisers N_int and N_bi, and the flat
buffer [dL/dtheta | alpha*L_pde | L_bi | nonfinite | pad] is summed by ONE allreduce
(torch.distributed; NCCL over NVLink/NVSwitch on the B200 box).  Adam then runs replicated on
every rank on bit-identical inputs, so parameters stay identical without a broadcast; the replica
check below verifies that (a digest of the parameters gathered from every rank).

`DPTrainStep` is the step bench.py times and the world_size-2 gloo tests run (with a CPU stub net
in place of HRKANNet, which exposes the same pinn_loss_grad / adam_step / get_params calls).
"""
from __future__ import annotations

import hashlib
from typing import Callable, Dict, Optional, Tuple

SET_KEYS = ("interior", "forcing", "boundary", "g_boundary", "initial", "g_initial")


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


def global_counts(sets: dict) -> Tuple[int, int]:
    """(N_int, N_bi) of the whole job: the loss normalisers every rank passes (DESIGN reading 13)."""
    n_int = 0 if sets.get("interior") is None else len(sets["interior"])
    n_bi = (0 if sets.get("boundary") is None else len(sets["boundary"])) + \
           (0 if sets.get("initial") is None else len(sets["initial"]))
    return n_int, n_bi


def dp_loss_grad(loss_grad_fn: Callable, sets: dict, rank: int, world: int, group=None,
                 allreduce: bool = True):
    """One data-parallel loss+grad evaluation.

    sets: {"interior", "forcing", "boundary", "g_boundary", "initial", "g_initial"} (full sets;
    each rank slices its shard here).  loss_grad_fn(interior=, forcing=, boundary=, g_boundary=,
    initial=, g_initial=, n_int_global=, n_bi_global=) -> flat buffer (torch tensor).
    Returns the allreduced buffer (identical on every rank)."""
    import torch.distributed as dist
    n_int, n_bi = global_counts(sets)
    local = {k: shard(v, rank, world) for k, v in sets.items()}
    out = loss_grad_fn(n_int_global=n_int, n_bi_global=n_bi, **local)
    if allreduce and world > 1:
        dist.all_reduce(out, op=dist.ReduceOp.SUM, group=group)
    return out


class DPTrainStep:
    """One data-parallel training step: pinn_loss_grad on this rank's shard (global normalisers)
    -> ONE all_reduce(SUM) of the flat [dtheta | loss parts | flag | pad] buffer -> replicated Adam.

    net:    HRKANNet (or any object with pinn_loss_grad(pde, interior, boundary, g_boundary, initial,
            g_initial, forcing=, n_int_global=, n_bi_global=, out=), adam_step(grad, lr=...), n_params)
    shard_sets: this rank's blocks (device tensors for the device-resident path; pinned host tensors
            for the end-to-end path can be passed per call)
    n_int_global, n_bi_global: the job's normalisers; out: the flat buffer (device tensor)."""

    def __init__(self, net, pde, shard_sets: Dict[str, object], n_int_global: int, n_bi_global: int, out,
                 world: int = 1, group=None, lr: float = 1e-3):
        self.net, self.pde, self.sets = net, pde, dict(shard_sets)
        self.n_int_global, self.n_bi_global = n_int_global, n_bi_global
        self.out, self.world, self.group, self.lr = out, world, group, lr
        self.npar = net.n_params

    def loss_grad(self, sets: Optional[Dict[str, object]] = None):
        s = self.sets if sets is None else sets
        self.net.pinn_loss_grad(self.pde, s["interior"], s["boundary"], s["g_boundary"], s.get("initial"),
                                s.get("g_initial"), forcing=s.get("forcing"), n_int_global=self.n_int_global,
                                n_bi_global=self.n_bi_global, out=self.out)
        if self.world > 1:
            import torch.distributed as dist
            dist.all_reduce(self.out, op=dist.ReduceOp.SUM, group=self.group)
        return self.out

    def __call__(self, sets: Optional[Dict[str, object]] = None, result=None):
        """One step; `result` (e.g. a pinned host tensor of 4 floats) receives [alpha L_pde, L_bi,
        flag, pad] asynchronously (the end-to-end path's device->host read)."""
        out = self.loss_grad(sets)
        self.net.adam_step(out[:self.npar], lr=self.lr)
        if result is not None:
            result.copy_(out[self.npar:self.npar + 4], non_blocking=True)
        return out


def params_digest(net) -> str:
    """sha256 of the flat fp32 parameter bytes (synchronising read)."""
    p = net.get_params()
    arr = p.detach().cpu().contiguous().numpy() if hasattr(p, "detach") else p
    return hashlib.sha256(arr.tobytes()).hexdigest()


def check_replicas(net, world: int, group=None) -> Tuple[bool, list]:
    """Gather every rank's parameter digest; (all equal, digests).  SURVEY §8(e): replicated Adam must
    keep bit-identical parameters (checked after init and after the timed steps)."""
    d = params_digest(net)
    if world <= 1:
        return True, [d]
    import torch.distributed as dist
    digests = [None] * world
    dist.all_gather_object(digests, d, group=group)
    return all(x == digests[0] for x in digests), digests
