"""GPU parity of SURVEY §8(f) row 3 -- higher-order and mixed jets -- against the float64 oracle of
oracle/hrkan_oracle_jets.py (a different derivation: truncated power-series composition, exact polynomial
basis derivatives, torch.autograd gradients) on identical seeded inputs, through the C ABI.

Tolerances (relative L2 over each tensor): u 1e-4, first derivatives 5e-4, second derivatives, loss and
every dW_l / db_l 2e-3 (BASELINE.json north_star); third to fifth x-derivatives JET_TOL below (DESIGN.md
"Higher-order jets: tolerances")."""
import numpy as np
import pytest

import hrkan_inputs as HI
from oracle import hrkan_oracle as O2
from oracle import hrkan_oracle_jets as OJ
from test_gpu_parity import rel_l2

pytestmark = pytest.mark.gpu

TOL = {"u": 1e-4, "d1": 5e-4, "d2": 2e-3, "loss": 2e-3, "grad": 2e-3}
JET_TOL = {3: 5e-3, 4: 1e-2, 5: 2e-2}


@pytest.fixture(scope="module")
def torch_mod():
    import torch
    assert torch.cuda.is_available()
    return torch


def _make(w, seed=7, bias_std=0.1, chunk=None):
    from paper_2409_14248_b200 import HRKANNet
    net = HRKANNet(w.widths, w.G, w.k, w.m, w.lo, w.hi)
    params = HI.random_params(w.widths, w.G, w.k, seed=seed, bias_std=bias_std)
    net.set_params(HI.flatten_params(params))
    if chunk:
        net.set_chunk_points(chunk)
    return net, params


def _pde(w):
    if w.pde == "kawahara":
        return {"kind": "kawahara", "alpha": w.alpha, "adv": w.adv, "disp3": w.disp3, "disp5": w.disp5}
    return {"kind": "aniso", "alpha": w.alpha, "K": list(w.aniso)}


def _pde_struct(w):
    from paper_2409_14248_b200 import pde_struct
    if w.pde == "kawahara":
        return pde_struct("kawahara", w.alpha, adv=w.adv, disp3=w.disp3, disp5=w.disp5)
    return pde_struct("aniso", w.alpha, aniso=list(w.aniso))


@pytest.mark.parametrize("m", [3, 6, 8])
def test_taylor5_jet_parity(torch_mod, m):
    """u, d^r u/dx^r (r = 1..5) and u_t of a [2,16,16,1] net (K1 shape) vs the oracle; m = 6 is the paper's
    choice for u_xxxxx, m = 3 the smallest order with a non-zero fifth derivative."""
    torch = torch_mod
    from paper_2409_14248_b200 import JET_TAYLOR5
    w = HI.WORKLOADS["K1"]
    w = HI.Workload(**{**w.__dict__, "m": m})
    net, params = _make(w, chunk=1500)                  # several chunks + a ragged tail
    pts = HI.make_points(w).interior[:3000]
    jet = net.forward_jet_ex(JET_TAYLOR5, torch.from_numpy(pts).cuda()).cpu().numpy()
    ux, ut = OJ.forward_taylor(OJ.Net(w.widths, w.G, w.k, m, w.lo, w.hi), OJ.params_to_torch(params), pts, 5)
    ux, ut = ux.numpy(), ut.numpy()
    errs = [rel_l2(jet[:, r], ux[:, r]) for r in range(6)] + [rel_l2(jet[:, 6], ut)]
    tol = [TOL["u"], TOL["d1"], TOL["d2"], JET_TOL[3], JET_TOL[4], JET_TOL[5], TOL["d1"]]
    assert all(e < t for e, t in zip(errs, tol)), (errs, tol)


@pytest.mark.parametrize("key", ["A2", "A3"])
def test_hessian_jet_parity(torch_mod, key):
    """u, grad u and the full Hessian (mixed terms included) vs the oracle; the diagonal also equals the
    library's own diagonal jet (hrkan_forward_jet), an independent kernel family."""
    torch = torch_mod
    from paper_2409_14248_b200 import JET_HESSIAN
    w = HI.WORKLOADS[key]
    D = w.D
    net, params = _make(w, chunk=1100)
    pts = HI.make_points(w).interior[:2500]
    jet = net.forward_jet_ex(JET_HESSIAN, torch.from_numpy(pts).cuda()).cpu().numpy()
    u, g, H = OJ.forward_hessian(OJ.Net(w.widths, w.G, w.k, w.m, w.lo, w.hi), OJ.params_to_torch(params), pts)
    pairs = OJ.pair_index(D)
    Hq = np.stack([H[:, a, b].numpy() for a, b in pairs], 1)
    assert rel_l2(jet[:, 0], u.numpy()) < TOL["u"]
    assert rel_l2(jet[:, 1:1 + D], g.numpy()) < TOL["d1"]
    assert rel_l2(jet[:, 1 + D:], Hq) < TOL["d2"]
    mixed = [q for q, (a, b) in enumerate(pairs) if a != b]
    assert rel_l2(jet[:, 1 + D + np.array(mixed)], Hq[:, mixed]) < TOL["d2"]
    u2, du2, d2u2 = [t.cpu().numpy() for t in net.forward_jet(torch.from_numpy(pts).cuda())]
    diag = [q for q, (a, b) in enumerate(pairs) if a == b]
    assert rel_l2(jet[:, 1 + D + np.array(diag)], d2u2) < 1e-5
    assert rel_l2(jet[:, 0], u2) < 1e-6


def _loss_grad_gpu(torch, net, w, ps, **kw):
    cu = lambda a: None if a is None else torch.from_numpy(a).cuda()
    out = net.pinn_loss_grad(_pde_struct(w), cu(ps.interior), cu(ps.boundary), cu(ps.g_boundary), cu(ps.initial),
                             cu(ps.g_initial), forcing=cu(ps.forcing), **kw)
    torch.cuda.synchronize()
    return out.cpu().numpy()


def _loss_grad_oracle(w, params, ps):
    bi = ps.boundary if ps.initial is None else np.concatenate([ps.boundary, ps.initial])
    gbi = ps.g_boundary if ps.initial is None else np.concatenate([ps.g_boundary, ps.g_initial])
    net = OJ.Net(w.widths, w.G, w.k, w.m, w.lo, w.hi)
    return OJ.loss_grad(net, [(W.astype(np.float64), b.astype(np.float64)) for W, b in params], _pde(w),
                        ps.interior, bi, gbi, forcing=ps.forcing)


def _check(out, w, lp, lb, g):
    npar = w.num_params()
    assert out[npar + 2] == 0.0
    assert abs(out[npar] - lp) <= TOL["loss"] * abs(lp) + 1e-12, (out[npar], lp)
    assert abs(out[npar + 1] - lb) <= TOL["loss"] * abs(lb) + 1e-12, (out[npar + 1], lb)
    flat = OJ.flat_grad(g)
    assert rel_l2(out[:npar], flat) < TOL["grad"]
    for l, ((gW, gb), (oW, ob)) in enumerate(zip(HI.unflatten_params(out[:npar].copy(), w.widths, w.B), g)):
        assert rel_l2(gW, oW) < TOL["grad"], f"dW layer {l}: {rel_l2(gW, oW)}"
        assert rel_l2(gb, ob) < TOL["grad"], f"db layer {l}: {rel_l2(gb, ob)}"


@pytest.mark.parametrize("key", ["K1", "A2", "A3"])
def test_loss_grad_parity(torch_mod, key):
    """Kawahara (u_xxxxx, m = 6) and anisotropic (mixed u_ab) loss + gradient vs the oracle on the full
    parity sets, chunked so several chunks and a ragged tail run."""
    torch = torch_mod
    w = HI.WORKLOADS[key]
    ps = HI.make_points(w)
    net, params = _make(w, chunk=1000)
    out = _loss_grad_gpu(torch, net, w, ps)
    _check(out, w, *_loss_grad_oracle(w, params, ps))


def test_k6_bench_shape_sampled(torch_mod):
    """The bench workload's net ([2,64,64,1], G=10, m=6) on a strided subset at the default chunking:
    loss + gradient parity, and the full-size Taylor jet on sampled points."""
    torch = torch_mod
    from paper_2409_14248_b200 import JET_TAYLOR5
    w = HI.WORKLOADS["K6"]
    ps = HI.make_points(w)
    sub = ps.subset(512, 16)
    net, params = _make(w)
    out = _loss_grad_gpu(torch, net, w, sub)
    _check(out, w, *_loss_grad_oracle(w, params, sub))
    jet = net.forward_jet_ex(JET_TAYLOR5, torch.from_numpy(ps.interior).cuda()).cpu().numpy()
    idx = np.random.default_rng(0).choice(len(ps.interior), 256, replace=False)
    ux, ut = OJ.forward_taylor(OJ.Net(w.widths, w.G, w.k, w.m), OJ.params_to_torch(params), ps.interior[idx], 5)
    assert rel_l2(jet[idx, 0], ux[:, 0].numpy()) < TOL["u"]
    assert rel_l2(jet[idx, 5], ux[:, 5].numpy()) < JET_TOL[5]
    assert rel_l2(jet[idx, 6], ut.numpy()) < TOL["d1"]
    assert np.isfinite(jet).all()


def test_jet_engine_invalid_arguments_and_shards(torch_mod):
    torch = torch_mod
    from paper_2409_14248_b200 import HRKANNet, HrkanError, JET_HESSIAN, JET_TAYLOR5, pde_struct
    w = HI.WORKLOADS["K1"]
    net2 = HRKANNet([2, 8, 1], 5, 3, 2)
    with pytest.raises(HrkanError):                       # u_xxxxx needs m >= 3
        net2.forward_jet_ex(JET_TAYLOR5, torch.zeros(4, 2, device="cuda"))
    with pytest.raises(HrkanError):
        net2.pinn_loss_grad(pde_struct("kawahara", disp3=0.01, disp5=1e-4), torch.zeros(4, 2, device="cuda"),
                            torch.zeros(0, 2, device="cuda"), torch.zeros(0, device="cuda"))
    with pytest.raises(HrkanError):                       # anisotropic operator without a forcing
        net2.pinn_loss_grad(pde_struct("aniso", aniso=[1, 0, 1]), torch.zeros(4, 2, device="cuda"),
                            torch.zeros(0, 2, device="cuda"), torch.zeros(0, device="cuda"))
    net3 = HRKANNet([3, 8, 1], 5, 3, 4)
    with pytest.raises(HrkanError):                       # Taylor-5 jet is (x, t) only
        net3.forward_jet_ex(JET_TAYLOR5, torch.zeros(4, 3, device="cuda"))
    assert net3.forward_jet_ex(JET_HESSIAN, torch.zeros(0, 3, device="cuda")).shape == (0, 10)
    # data-parallel shards with global normalisers sum to the unsharded call (generic engine)
    ps = HI.make_points(w)
    net, _ = _make(w)
    full = _loss_grad_gpu(torch, net, w, ps)
    acc = np.zeros_like(full, dtype=np.float64)
    for r in range(3):
        acc += _loss_grad_gpu(torch, net, w, ps.shard(r, 3), n_int_global=len(ps.interior), n_bi_global=ps.n_bi)
    assert rel_l2(acc, full) < 1e-5
    # run-to-run bitwise determinism
    np.testing.assert_array_equal(_loss_grad_gpu(torch, net, w, ps), full)
