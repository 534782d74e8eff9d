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


# ------------------------------------------------------------------ bench.py's own DP step and launcher
def _dp_step_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        from paper_2409_14248_b200.parallel import DPTrainStep, check_replicas, global_counts
        w = HI.WORKLOADS["C2"]
        ps = HI.make_points(w).subset(7, 3)
        sh = ps.shard(rank, world)
        n_int, n_bi = global_counts({"interior": ps.interior, "boundary": ps.boundary, "initial": ps.initial})
        net = bench.StubNet(2, seed=1)
        t = lambda a: None if a is None else torch.from_numpy(a)
        sets = {"interior": t(sh.interior), "boundary": t(sh.boundary), "g_boundary": t(sh.g_boundary),
                "initial": t(sh.initial), "g_initial": t(sh.g_initial)}
        out = torch.empty(net.n_params + 4)
        step = DPTrainStep(net, None, sets, n_int, n_bi, out, world=world, lr=1e-2)
        same0, _ = check_replicas(net, world)
        grads = []
        for _ in range(3):
            grads.append(step().clone().numpy())
        same1, dig = check_replicas(net, world)
        q.put((rank, same0, same1, grads, net.get_params().numpy()))
    finally:
        dist.destroy_process_group()


def test_dp_train_step_world2_matches_single_process():
    """DPTrainStep (the step bench.py times): 2 gloo ranks with a CPU stub net give the same allreduced
    buffers and post-Adam parameters as one process over the whole set, and the replica digests agree."""
    from bench import StubNet
    from paper_2409_14248_b200.parallel import DPTrainStep
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dp_step_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {r: rest for r, *rest in (q.get(timeout=300) for _ in range(world))}
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        assert res[r][0] and res[r][1]                     # identical params after init and after steps
    np.testing.assert_array_equal(res[0][3], res[1][3])
    # single process over the whole set
    w = HI.WORKLOADS["C2"]
    ps = HI.make_points(w).subset(7, 3)
    net = StubNet(2, seed=1)
    t = lambda a: None if a is None else torch.from_numpy(a)
    sets = {"interior": t(ps.interior), "boundary": t(ps.boundary), "g_boundary": t(ps.g_boundary),
            "initial": t(ps.initial), "g_initial": t(ps.g_initial)}
    out = torch.empty(net.n_params + 4)
    step = DPTrainStep(net, None, sets, len(ps.interior), ps.n_bi, out, world=1, lr=1e-2)
    for i in range(3):
        g = step().clone().numpy()
        np.testing.assert_allclose(res[0][2][i], g, rtol=2e-5, atol=1e-6)
    np.testing.assert_allclose(res[0][3], net.get_params().numpy(), rtol=2e-5, atol=1e-6)


def test_bench_launcher_dry_run_two_ranks():
    """`bench.py --gpus 2 --dry-run` (no WORLD_SIZE): the launcher builds once, re-executes itself under
    torch.distributed.run with 2 ranks (gloo + stub net on CPU), and rank 0 prints ONE JSON line with
    n_gpus 2, one build in total, and bit-identical parameters on both ranks after the steps."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "HRKAN_BENCH_BUILT")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--dry-run", "--steps", "2",
                        "--warmup", "1", "--config", "C2"], capture_output=True, text=True, timeout=600, env=env,
                       cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["comm"]["world_size"] == 2 and d["config"]["parallelism"] == "dp2"
    assert d["builds"]["total"] == 1 and d["builds"]["per_rank"] == [0, 0]
    assert d["replicas"]["params_identical_after_init"] and d["replicas"]["params_identical_after_steps"]
    assert d["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
