"""World-size-2 data-parallel host logic on CPU (gloo): each rank evaluates its contiguous point
shard with the global normalisers and ONE allreduce of the flat buffer reproduces the
unsharded loss and gradient.  The per-rank evaluation is the float64 oracle
here (no GPU in CI); on the B200 box it is HRKANNet.pinn_loss_grad."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import hrkan_inputs as HI
from oracle import hrkan_oracle as O
from paper_2409_14248_b200.parallel import dp_loss_grad, shard_range

BURGERS = {"kind": "burgers", "alpha": 0.05, "adv": 1.0, "visc": 0.01 / np.pi}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem():
    w = HI.WORKLOADS["C2"]
    ps = HI.make_points(w).subset(25, 8)
    net = O.Net(w.widths, w.G, w.k, w.m)
    params = HI.random_params(w.widths, w.G, w.k, seed=5, bias_std=0.1)
    sets = {"interior": ps.interior, "forcing": None, "boundary": ps.boundary, "g_boundary": ps.g_boundary,
            "initial": ps.initial, "g_initial": ps.g_initial}
    return net, params, sets


def _oracle_fn(net, params):
    def fn(interior, forcing, boundary, g_boundary, initial, g_initial, n_int_global, n_bi_global):
        bi = np.concatenate([boundary, initial])
        gbi = np.concatenate([g_boundary, g_initial])
        lp, lb, g = O.loss_grad(net, params, BURGERS, interior, bi, gbi, n_int_global=n_int_global,
                                n_bi_global=n_bi_global)
        return torch.from_numpy(np.concatenate([O.flat_grad(g), [lp, lb, 0.0, 0.0]]))
    return fn


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        net, params, sets = _problem()
        out = dp_loss_grad(_oracle_fn(net, params), sets, rank, world)
        q.put((rank, out.numpy()))
    finally:
        dist.destroy_process_group()


def test_shard_range_partition():
    for n in [0, 1, 7, 100, 2 ** 20 + 3]:
        for world in [1, 2, 3, 8]:
            blocks = [shard_range(n, r, world) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            assert all(blocks[r][1] == blocks[r + 1][0] for r in range(world - 1))
            sizes = [b - a for a, b in blocks]
            assert max(sizes) - min(sizes) <= 1


def test_gloo_world2_matches_unsharded():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    net, params, sets = _problem()
    ref = _oracle_fn(net, params)(n_int_global=len(sets["interior"]),
                                  n_bi_global=len(sets["boundary"]) + len(sets["initial"]), **sets).numpy()
    np.testing.assert_array_equal(res[0], res[1])          # identical on every rank
    np.testing.assert_allclose(res[0], ref, rtol=1e-10, atol=1e-14)
