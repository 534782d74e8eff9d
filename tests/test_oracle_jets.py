"""Pins of oracle/hrkan_oracle_jets.py (higher-order and mixed jets) against what the
paper and mathematics fix: sympy-exact basis derivatives of Eq. 2 to order 8 and the continuity class
C^{m-1}, exact polynomial nets (fifth-order and mixed second-order derivatives through one and
two layers), finite differences, the exact Kawahara solitary wave, a manufactured anisotropic solution,
the order-2 channels against the independent numpy oracle, and finite-difference gradients."""
import numpy as np
import pytest
import sympy as sp
import torch

import hrkan_inputs as HI
from oracle import hrkan_oracle as O2
from oracle import hrkan_oracle_jets as OJ



def _sym_basis(m, s, e, xs):
    return (2 / (e - s)) ** (2 * m) * ((e - xs) * (xs - s)) ** m


@pytest.mark.parametrize("m", [2, 4, 6, 7, 8])
def test_basis_all_orders_vs_sympy(m):
    """v^{(d)}, d = 0..8, at rational points of two supports: exact Eq. 2 differentiated by sympy."""
    xs = sp.symbols("x")
    G, k, lo, hi = 5, 3, -1, 1
    s, e = OJ.make_supports(G, k, lo, hi)
    h = sp.Rational(hi - lo, G)
    for n in (2, 6):
        sn = lo + (n - k) * h
        en = sn + (k + 1) * h
        v = _sym_basis(m, sn, en, xs)
        pts = [sn + (en - sn) * sp.Rational(q, 17) for q in (1, 5, 8, 13, 16)]
        xt = torch.tensor([float(p) for p in pts], dtype=torch.float64)
        for d in range(9):
            got = OJ.basis(xt, s, e, m, d)[:, n].numpy()
            ref = np.array([float(sp.diff(v, xs, d).subs(xs, p)) for p in pts])
            scale = max(1.0, np.abs(ref).max())
            np.testing.assert_allclose(got, ref, rtol=1e-10, atol=1e-10 * scale)


@pytest.mark.parametrize("m", [3, 5, 6])
def test_basis_continuity_class(m):
    """C^{m-1}: derivatives of order < m tend to 0 at the support's ends (one-sided limits from
    inside match the zero outside); order m jumps to the sympy value; outside the support every order is 0."""
    s, e = OJ.make_supports(5, 3, -1.0, 1.0)
    n = 4
    eps = 1e-7 * (e[n] - s[n])
    x_in = torch.tensor([s[n] + eps, e[n] - eps], dtype=torch.float64)
    x_out = torch.tensor([s[n] - eps, e[n] + eps, s[n], e[n]], dtype=torch.float64)
    xs = sp.symbols("x")
    v = _sym_basis(m, sp.nsimplify(s[n]), sp.nsimplify(e[n]), xs)
    for d in range(m + 2):
        inside = OJ.basis(x_in, s, e, m, d)[:, n].numpy()
        assert np.all(OJ.basis(x_out, s, e, m, d)[:, n].numpy() == 0.0)
        lim = float(sp.diff(v, xs, d).subs(xs, sp.nsimplify(s[n])))
        grid = torch.linspace(s[n], e[n], 401, dtype=torch.float64)[1:-1]
        scale = OJ.basis(grid, s, e, m, d)[:, n].abs().max().item()
        if d < m:
            assert lim == 0.0 and np.all(np.abs(inside) < 1e-4 * scale)
        elif d == m:
            assert lim != 0.0 and inside[0] == pytest.approx(lim, rel=1e-5)


def _p_setup():
    """P2-style chain through one neuron per layer on a rational grid: u = v_{n'}(z), z = lam (v_n(x) + v_n(t)) + b0."""
    G, k, lo, hi = 5, 3, -1, 1
    B = G + k
    s, e = OJ.make_supports(G, k, lo, hi)
    nstar, nprime = 3, 4
    w = e[0] - s[0]
    lam, b0 = w / 4, s[nprime] + w / 8
    W0 = np.zeros((1, 2, B)); W0[0, 0, nstar] = lam; W0[0, 1, nstar] = lam
    W1 = np.zeros((1, 1, B)); W1[0, 0, nprime] = 1.0
    params = [(W0, np.array([b0])), (W1, np.array([0.0]))]
    return (G, k, lo, hi, B, nstar, nprime, lam, b0), params


@pytest.mark.parametrize("m", [3, 6])
def test_taylor_jet_exact_two_layer_chain(m):
    """u = v_{n'}(lam (v_n(x) + v_n(t)) + b0): d^r u/dx^r for r = 0..5 and du/dt against sympy."""
    (G, k, lo, hi, B, nstar, nprime, lam, b0), params = _p_setup()
    net = OJ.Net([2, 1, 1], G, k, m, lo, hi)
    x, t = sp.symbols("x t")
    h = sp.Rational(hi - lo, G)
    sn = lo + (nstar - k) * h
    en = sn + (k + 1) * h
    sp_ = lo + (nprime - k) * h
    ep_ = sp_ + (k + 1) * h
    z = sp.nsimplify(lam) * (_sym_basis(m, sn, en, x) + _sym_basis(m, sn, en, t)) + sp.nsimplify(b0)
    u = _sym_basis(m, sp_, ep_, z)
    rng = np.random.default_rng(0)
    P = np.stack([rng.uniform(float(sn) + 0.02, float(en) - 0.02, 6), rng.uniform(float(sn) + 0.02, float(en) - 0.02, 6)], 1)
    ux, ut = OJ.forward_taylor(net, OJ.params_to_torch(params), P, 5)
    for q in range(len(P)):
        sub = {x: sp.nsimplify(P[q, 0]), t: sp.nsimplify(P[q, 1])}
        for r in range(6):
            ref = float(sp.diff(u, x, r).subs(sub))
            assert ux[q, r].item() == pytest.approx(ref, rel=1e-9, abs=1e-9 * max(1, abs(ref)))
        assert ut[q].item() == pytest.approx(float(sp.diff(u, t).subs(sub)), rel=1e-9, abs=1e-12)


@pytest.mark.parametrize("m", [2, 4, 6])
def test_hessian_exact_two_layer_chain(m):
    """Mixed second derivatives u_xy of the same chain (d2u symmetric, all entries) vs sympy."""
    (G, k, lo, hi, B, nstar, nprime, lam, b0), params = _p_setup()
    net = OJ.Net([2, 1, 1], G, k, m, lo, hi)
    x, y = sp.symbols("x y")
    h = sp.Rational(hi - lo, G)
    sn = lo + (nstar - k) * h
    en = sn + (k + 1) * h
    sp_ = lo + (nprime - k) * h
    ep_ = sp_ + (k + 1) * h
    z = sp.nsimplify(lam) * (_sym_basis(m, sn, en, x) + _sym_basis(m, sn, en, y)) + sp.nsimplify(b0)
    u = _sym_basis(m, sp_, ep_, z)
    rng = np.random.default_rng(1)
    P = rng.uniform(float(sn) + 0.02, float(en) - 0.02, (5, 2))
    uu, g, H = OJ.forward_hessian(net, OJ.params_to_torch(params), P)
    for q in range(len(P)):
        sub = {x: sp.nsimplify(P[q, 0]), y: sp.nsimplify(P[q, 1])}
        for (a, va), (b, vb) in [((0, x), (0, x)), ((0, x), (1, y)), ((1, y), (1, y))]:
            ref = float(sp.diff(u, va, vb).subs(sub))
            assert H[q, a, b].item() == pytest.approx(ref, rel=1e-9, abs=1e-9 * max(1, abs(ref)))
            assert H[q, b, a].item() == pytest.approx(H[q, a, b].item(), rel=1e-13, abs=1e-15)
        assert g[q, 1].item() == pytest.approx(float(sp.diff(u, y).subs(sub)), rel=1e-9, abs=1e-12)


def _rand(widths, G=6, k=3, m=6, seed=0, lo=-1.0, hi=1.0):
    net = OJ.Net(widths, G, k, m, lo, hi)
    params = HI.random_params(widths, G, k, seed=seed, bias_std=0.2)
    return net, [(W.astype(np.float64), b.astype(np.float64)) for W, b in params]


def test_taylor_jet_finite_differences():
    """Each order is the derivative of the previous one along x (central FD of order r-1 at +-h), on a
    random [2,4,3,1] m = 6 net; the t channel is the FD of u along t."""
    net, params = _rand([2, 4, 3, 1], seed=3)
    pt = OJ.params_to_torch(params)
    P = np.random.default_rng(2).uniform(-0.9, 0.9, (40, 2))
    h = 1e-5
    ux, ut = OJ.forward_taylor(net, pt, P, 5)
    up, _ = OJ.forward_taylor(net, pt, P + [h, 0], 5)
    um, _ = OJ.forward_taylor(net, pt, P - [h, 0], 5)
    for r in range(1, 6):
        fd = (up[:, r - 1] - um[:, r - 1]) / (2 * h)
        scale = ux[:, r].abs().max().item()
        assert (fd - ux[:, r]).abs().max().item() < 1e-5 * scale
    vp, _ = OJ.forward_taylor(net, pt, P + [0, h], 5)
    vm, _ = OJ.forward_taylor(net, pt, P - [0, h], 5)
    fd = (vp[:, 0] - vm[:, 0]) / (2 * h)
    assert (fd - ut).abs().max().item() < 1e-6 * ut.abs().max().item()


def test_hessian_finite_differences_3d():
    net, params = _rand([3, 3, 2, 1], m=4, seed=4)
    pt = OJ.params_to_torch(params)
    P = np.random.default_rng(3).uniform(-0.9, 0.9, (30, 3))
    u, g, H = OJ.forward_hessian(net, pt, P)
    h = 1e-5
    for a in range(3):
        e = np.zeros(3); e[a] = h
        _, gp, _ = OJ.forward_hessian(net, pt, P + e)
        _, gm, _ = OJ.forward_hessian(net, pt, P - e)
        fd = (gp - gm) / (2 * h)                              # fd[p, b] = d/dxi_a du/dxi_b
        assert (fd - H[:, a, :]).abs().max().item() < 1e-5 * H.abs().max().item()
    np.testing.assert_allclose(H.numpy(), np.transpose(H.numpy(), (0, 2, 1)), rtol=0, atol=1e-14)


@pytest.mark.parametrize("widths,m", [([2, 4, 3, 1], 4), ([3, 3, 1], 6)])
def test_order2_channels_match_numpy_oracle(widths, m):
    """Independent derivations agree: the Taylor jet's u, u_x, u_xx and the Hessian's gradient and diagonal
    equal hrkan_oracle.forward_jet (numpy, closed-form p-form derivatives, diagonal chain rule)."""
    net, params = _rand(widths, m=m, seed=5)
    net2 = O2.Net(widths, 6, 3, m)
    P = np.random.default_rng(4).uniform(-0.95, 0.95, (50, widths[0]))
    u2, du2, d2u2 = O2.forward_jet(net2, params, P)
    pt = OJ.params_to_torch(params)
    u, g, H = OJ.forward_hessian(net, pt, P)
    np.testing.assert_allclose(u.numpy(), u2, rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(g.numpy(), du2, rtol=1e-11, atol=1e-12)
    np.testing.assert_allclose(np.diagonal(H.numpy(), axis1=1, axis2=2), d2u2, rtol=1e-10, atol=1e-11)
    if widths[0] == 2:
        ux, ut = OJ.forward_taylor(net, pt, P, 2)
        np.testing.assert_allclose(ux[:, 0].numpy(), u2, rtol=1e-12, atol=1e-13)
        np.testing.assert_allclose(ux[:, 1].numpy(), du2[:, 0], rtol=1e-11, atol=1e-12)
        np.testing.assert_allclose(ux[:, 2].numpy(), d2u2[:, 0], rtol=1e-10, atol=1e-11)
        np.testing.assert_allclose(ut.numpy(), du2[:, 1], rtol=1e-11, atol=1e-12)


def test_kawahara_residual_exact_solitary_wave():
    """The exact solitary wave of u_t + a u u_x + b u_xxx - c u_xxxxx = 0,
    u = (105 b^2 / (169 a c)) sech^4( sqrt(b / (13 c)) / 2 (x - 36 b^2 t / (169 c)) ), gives a zero residual
    while every term is non-zero (a flipped sign or a wrong order of any term fails)."""
    a, b, c = 1.0, 0.01, 1e-4
    x, t = sp.symbols("x t")
    A = 105 * b ** 2 / (169 * a * c)
    kap = sp.sqrt(b / (13 * c)) / 2
    V = 36 * b ** 2 / (169 * c)
    u = A * sp.sech(kap * (x - V * t)) ** 4
    f = sp.lambdify((x, t), [sp.diff(u, x, r) for r in range(6)] + [sp.diff(u, t)], "numpy")
    P = np.random.default_rng(7).uniform(-1, 1, (40, 2))
    P[:, 1] = np.abs(P[:, 1])
    vals = [np.asarray(v, np.float64) * np.ones(len(P)) for v in f(P[:, 0], P[:, 1])]
    ux = torch.tensor(np.stack(vals[:6], 1))
    ut = torch.tensor(vals[6])
    r = OJ.kawahara_residual(ux[:, 0], ux, ut, a, b, c)
    terms = [ut, a * ux[:, 0] * ux[:, 1], b * ux[:, 3], c * ux[:, 5]]
    scale = sum(tt.abs() for tt in terms)
    assert (r.abs() <= 1e-10 * scale).all()
    for tt in terms:
        assert tt.abs().max() > 1e-3 * scale.max()
    wrong = ut + a * ux[:, 0] * ux[:, 1] + b * ux[:, 3] + c * ux[:, 5]
    assert (wrong.abs() / scale).max() > 1e-2


def test_aniso_residual_manufactured_solution():
    """u* = prod_a sin(pi x_a) with f = sum_{a<=b} K_ab d_a d_b u*: residual 0; K = identity (diagonal
    pairs) and f = the Poisson forcing reduces to the Poisson residual of hrkan_oracle."""
    rng = np.random.default_rng(8)
    for D in (2, 3):
        pairs = OJ.pair_index(D)
        P = rng.uniform(-1, 1, (30, D))
        s = np.sin(np.pi * P)
        cth = np.cos(np.pi * P)
        H = np.zeros((30, D, D))
        for a in range(D):
            for b in range(D):
                if a == b:
                    H[:, a, a] = -np.pi ** 2 * np.prod(s, 1)
                else:
                    rest = np.prod(np.delete(s, [a, b], axis=1), 1) if D > 2 else 1.0
                    H[:, a, b] = np.pi ** 2 * cth[:, a] * cth[:, b] * rest
        K = rng.uniform(-1, 1, len(pairs))
        f = sum(K[q] * H[:, a, b] for q, (a, b) in enumerate(pairs))
        r = OJ.aniso_residual(torch.tensor(H), K, f)
        assert r.abs().max() < 1e-12
        Kid = [1.0 if a == b else 0.0 for a, b in pairs]
        fP = O2.poisson_forcing(P)
        r2 = OJ.aniso_residual(torch.tensor(H), Kid, fP)
        ref = O2.poisson_residual(None, np.diagonal(H, axis1=1, axis2=2), P)
        np.testing.assert_allclose(r2.numpy(), ref, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("kind", ["kawahara", "aniso2", "aniso3"])
def test_gradient_vs_central_fd(kind):
    """dL/dtheta (torch.autograd, float64) vs central finite differences on 25 random parameters."""
    if kind == "kawahara":
        widths, m = [2, 3, 2, 1], 6
        pde = {"kind": "kawahara", "alpha": 0.05, "adv": 1.0, "disp3": 0.01, "disp5": 1e-4}
    else:
        D = 2 if kind == "aniso2" else 3
        widths, m = [D, 3, 1], 4
        pde = {"kind": "aniso", "alpha": 0.05, "K": list(np.linspace(0.3, 1.2, len(OJ.pair_index(D))))}
    net, params = _rand(widths, m=m, seed=9)
    rng = np.random.default_rng(10)
    Pi = rng.uniform(-0.9, 0.9, (25, widths[0]))
    Pb = rng.uniform(-1, 1, (8, widths[0]))
    gb = rng.uniform(-0.3, 0.3, 8)
    f = rng.uniform(-1, 1, 25)
    lp, lb, g = OJ.loss_grad(net, params, pde, Pi, Pb, gb, forcing=f)
    gflat = OJ.flat_grad(g)
    flat = OJ.flat_grad(params)

    def L(fl):
        pr = HI.unflatten_params(fl, widths, net.B)
        a, b = OJ.loss_parts(net, OJ.params_to_torch(pr), pde, Pi, Pb, gb, forcing=f)
        return float(a + b)

    idx = rng.choice(len(flat), 25, replace=False)
    for q in idx:
        st = 1e-6 * max(1.0, abs(flat[q]))
        fp, fm = flat.copy(), flat.copy()
        fp[q] += st
        fm[q] -= st
        fd = (L(fp) - L(fm)) / (2 * st)
        assert abs(fd - gflat[q]) <= 1e-6 * max(abs(gflat[q]), 1e-3 * np.abs(gflat).max())
    assert lp + lb == pytest.approx(L(flat), rel=1e-14)
