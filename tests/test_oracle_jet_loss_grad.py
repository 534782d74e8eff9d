"""Pins of the oracle's forward jet, residuals, loss, reverse pass and Adam against sympy-exact
polynomial nets, finite differences, complex-step, closed forms and SPEC examples."""
import os
from fractions import Fraction

import numpy as np
import pytest
import sympy as sp

import hrkan_inputs as HI
from oracle import hrkan_oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
POISSON = {"kind": "poisson", "alpha": 0.05, "adv": 0.0, "visc": 0.0}
BURGERS = {"kind": "burgers", "alpha": 0.05, "adv": 1.0, "visc": 0.01 / np.pi}


def _zero_params(widths, B):
    return [(np.zeros((widths[l + 1], widths[l], B)), np.zeros(widths[l + 1])) for l in range(len(widths) - 1)]


# ---------------------------------------------------------------- polynomial nets (exact)
def _sym_v(n, G, k, m, lo, hi, arg):
    """Eq. 2 on the interior of support n, in exact rational arithmetic."""
    h = Fraction(hi - lo) / G if isinstance(lo, int) else None
    h = sp.Rational(hi - lo, G)
    s = lo + (n - k) * h
    e = s + (k + 1) * h
    c = (2 / (e - s)) ** (2 * m)
    return ((e - arg) * (arg - s)) ** m * c, s, e


@pytest.mark.parametrize("m", [2, 3, 4])
def test_P1_single_layer_exact(m):
    """P1: [2,1] with W[0,0,n*] = W[0,1,n*] = 1: u = v(x) + v(y), laplacian = v''(x) + v''(y)."""
    G, k, lo, hi = 5, 3, -1, 1
    nstar = 4
    x, y = sp.symbols("x y")
    vx, s, e = _sym_v(nstar, G, k, m, lo, hi, x)
    vy, _, _ = _sym_v(nstar, G, k, m, lo, hi, y)
    u = vx + vy
    net = O.Net([2, 1], G, k, m, lo, hi)
    W = np.zeros((1, 2, G + k))
    W[0, 0, nstar] = W[0, 1, nstar] = 1.0
    params = [(W, np.zeros(1))]
    pts = [(sp.Rational(1, 7), sp.Rational(-1, 3)), (sp.Rational(9, 10), sp.Rational(1, 2)), (sp.Rational(-1, 2), sp.Rational(3, 4))]
    P = np.array([[float(a), float(b)] for a, b in pts])
    uo, duo, d2uo = O.forward_jet(net, params, P)
    for q, (a, b) in enumerate(pts):
        sub = {x: a, y: b}
        assert uo[q] == pytest.approx(float(u.subs(sub)), rel=1e-13)
        assert duo[q, 0] == pytest.approx(float(sp.diff(u, x).subs(sub)), rel=1e-12, abs=1e-12)
        assert duo[q, 1] == pytest.approx(float(sp.diff(u, y).subs(sub)), rel=1e-12, abs=1e-12)
        assert d2uo[q, 0] == pytest.approx(float(sp.diff(u, x, 2).subs(sub)), rel=1e-12, abs=1e-12)
        assert d2uo[q, 1] == pytest.approx(float(sp.diff(u, y, 2).subs(sub)), rel=1e-12, abs=1e-12)


def _p2_setup(m, widths=(2, 1, 1), D=2, G=5, k=3):
    """P2/P3: a chain through neuron 0 of every layer; scale/offset keep every intermediate
    inside one support so u is a polynomial with an exactly computable laplacian."""
    lo, hi = -1, 1
    B = G + k
    h = sp.Rational(hi - lo, G)
    w = (k + 1) * h
    nstar, nprime = 4, 2
    syms = sp.symbols("x0:%d" % D)
    vs = [_sym_v(nstar, G, k, m, lo, hi, z)[0] for z in syms]
    s_np = lo + (nprime - k) * h
    lam = w / 4 / D * 2            # z in [b0, b0 + D*lam] = [s'+w/8, s'+w/8+w/2]
    b0 = s_np + w / 8
    z = lam * sum(vs) + b0
    params = []
    L = len(widths) - 1
    W0 = np.zeros((widths[1], D, B))
    W0[0, :, nstar] = float(lam)
    b0v = np.zeros(widths[1])
    b0v[0] = float(b0)
    params.append((W0, b0v))
    expr = z
    for l in range(1, L):
        vz = _sym_v(nprime, G, k, m, lo, hi, expr)[0]
        Wl = np.zeros((widths[l + 1], widths[l], B))
        bl = np.zeros(widths[l + 1])
        if l < L - 1:
            # next intermediate: lam2 * v(z) + b2 stays inside support n'
            Wl[0, 0, nprime] = float(w / 2)
            bl[0] = float(b0)
            expr = (w / 2) * vz + b0
        else:
            Wl[0, 0, nprime] = 1.0
            expr = vz
        params.append((Wl, bl))
    return syms, expr, params, (G, k, lo, hi)


@pytest.mark.parametrize("m", [2, 4])
@pytest.mark.parametrize("widths", [(2, 1, 1), (2, 4, 3, 1), (3, 4, 4, 1)])
def test_P2_P3_chain_exact_laplacian(m, widths):
    D = widths[0]
    syms, u, params, (G, k, lo, hi) = _p2_setup(m, widths, D)
    net = O.Net(list(widths), G, k, m, lo, hi)
    rng = np.random.default_rng(3)
    # rational points inside (s_{n*}, e_{n*})^D = (-3/5, 1)^D
    pts = [[sp.Rational(int(rng.integers(-59, 99)), 100) for _ in range(D)] for _ in range(3)]
    P = np.array([[float(a) for a in p] for p in pts])
    uo, duo, d2uo = O.forward_jet(net, params, P)
    lap_o = d2uo.sum(1)
    for q, p in enumerate(pts):
        sub = dict(zip(syms, p))
        ref_u = float(u.subs(sub))
        ref_lap = float(sum(sp.diff(u, z, 2) for z in syms).subs(sub))
        assert uo[q] == pytest.approx(ref_u, rel=1e-12)
        assert lap_o[q] == pytest.approx(ref_lap, rel=1e-9, abs=1e-9)
        for a, z in enumerate(syms):
            assert duo[q, a] == pytest.approx(float(sp.diff(u, z).subs(sub)), rel=1e-9, abs=1e-10)


# ---------------------------------------------------------------- jets vs FD / complex step
def _rand_net(widths, G=5, k=3, m=4, seed=0, bias_std=0.1):
    net = O.Net(widths, G, k, m)
    params = [(W.astype(np.float64), b.astype(np.float64))
              for W, b in HI.random_params(widths, G, k, seed=seed, bias_std=bias_std)]
    return net, params


@pytest.mark.parametrize("widths", [[2, 5, 1], [2, 5, 5, 1], [3, 6, 4, 1], [1, 3, 1]])
def test_jet_vs_fd(widths):
    """du, d2u match central finite differences of forward (step 1e-4), rel < 1e-5."""
    net, params = _rand_net(widths, seed=len(widths))
    D = widths[0]
    P = np.random.default_rng(1).uniform(-0.9, 0.9, (20, D))
    u, du, d2u = O.forward_jet(net, params, P)
    np.testing.assert_allclose(u, O.forward_value(net, params, P), rtol=1e-14, atol=1e-14)
    h = 1e-4
    for a in range(D):
        E = np.zeros(D)
        E[a] = h
        fp, f0, fm = (O.forward_value(net, params, P + E), O.forward_value(net, params, P),
                      O.forward_value(net, params, P - E))
        fd1 = (fp - fm) / (2 * h)
        fd2 = (fp - 2 * f0 + fm) / h ** 2
        assert np.linalg.norm(fd1 - du[:, a]) <= 1e-5 * np.linalg.norm(du[:, a])
        assert np.linalg.norm(fd2 - d2u[:, a]) <= 1e-5 * np.linalg.norm(d2u[:, a])
        # complex step: exact first derivative
        cs = np.imag(O.forward_value(net, params, P + 1j * 1e-30 * (np.arange(D) == a))) / 1e-30
        np.testing.assert_allclose(cs, du[:, a], rtol=1e-12, atol=1e-13)


def test_linearity_in_last_layer():
    """the output is linear in the last layer's coefficients (superposition)."""
    net, params = _rand_net([2, 5, 5, 1], seed=4, bias_std=0.0)
    P = np.random.default_rng(2).uniform(-1, 1, (16, 2))
    W1 = np.random.default_rng(5).standard_normal(params[-1][0].shape)
    W2 = np.random.default_rng(6).standard_normal(params[-1][0].shape)
    zb = np.zeros(1)
    j1 = O.forward_jet(net, params[:-1] + [(W1, zb)], P)
    j2 = O.forward_jet(net, params[:-1] + [(W2, zb)], P)
    j12 = O.forward_jet(net, params[:-1] + [(W1 + W2, zb)], P)
    for a, b, c in zip(j1, j2, j12):
        np.testing.assert_allclose(a + b, c, rtol=1e-12, atol=1e-12)


def test_zero_weights_zero_jet_except_bias():
    net = O.Net([2, 5, 1], 5, 3, 4)
    params = _zero_params([2, 5, 1], 8)
    params[-1] = (params[-1][0], np.array([0.7]))
    u, du, d2u = O.forward_jet(net, params, np.random.default_rng(0).uniform(-1, 1, (9, 2)))
    assert np.all(u == 0.7) and np.all(du == 0) and np.all(d2u == 0)


# ---------------------------------------------------------------- residuals and loss
def test_residual_examples():
    # u == 0 at (1/2, 1/2) gives Poisson residual 2 pi^2
    r = O.poisson_residual(np.zeros((1, 2)), np.zeros((1, 2)), np.array([[0.5, 0.5]]))
    assert r[0] == pytest.approx(2 * np.pi ** 2, rel=1e-15)
    # u == 0 at (0, y) gives 0
    assert O.poisson_residual(np.zeros((1, 2)), np.zeros((1, 2)), np.array([[0.0, 0.3]]))[0] == 0.0
    # u = t gives Burgers residual 1 (u_t = 1, rest 0)
    r = O.burgers_residual(np.array([0.0]), np.array([[0.0, 1.0]]), np.zeros((1, 2)), 1.0, 0.01 / np.pi)
    assert r[0] == 1.0
    # the exact Poisson solution sin(pi x) sin(pi y) has zero residual (analytic jet)
    P = np.random.default_rng(0).uniform(-1, 1, (100, 2))
    sx, sy = np.sin(np.pi * P[:, 0]), np.sin(np.pi * P[:, 1])
    d2 = np.stack([-np.pi ** 2 * sx * sy, -np.pi ** 2 * sx * sy], 1)
    assert np.abs(O.poisson_residual(None, d2, P)).max() < 1e-10


def test_zero_weight_loss_closed_forms():
    rows = [l.split() for l in open(os.path.join(GOLDEN, "zero_weight_losses.txt")) if not l.startswith("#")]
    assert rows
    for key, beta, ref in rows:
        w = HI.WORKLOADS[key]
        ps = HI.make_points(w)
        net = O.Net(w.widths, w.G, w.k, w.m)
        params = _zero_params(w.widths, w.B)
        params[-1] = (params[-1][0], np.array([float(beta)]))
        pde = POISSON if w.pde == "poisson" else BURGERS
        bi = ps.boundary if ps.initial is None else np.concatenate([ps.boundary, ps.initial])
        gbi = ps.g_boundary if ps.initial is None else np.concatenate([ps.g_boundary, ps.g_initial])
        L = O.loss(net, params, pde, ps.interior, bi, gbi)
        assert L == pytest.approx(float(ref), rel=2e-6)
        # alpha = 0  =>  L = L_bi
        L0 = O.loss(net, params, {**pde, "alpha": 0.0}, ps.interior, bi, gbi)
        lp, lb = O.loss_parts(net, params, pde, ps.interior, bi, gbi)
        assert L0 == pytest.approx(lb, rel=1e-15)


# ---------------------------------------------------------------- gradient
@pytest.mark.parametrize("pde", [POISSON, BURGERS])
@pytest.mark.parametrize("m", [4, 5])
def test_grad_complex_step_all_params(pde, m):
    """Every parameter of a [2,3,2,1] net: hand-written reverse pass == complex-step derivative
    (machine precision).  Complex-step differentiates the forward loss only."""
    widths = [2, 3, 2, 1]
    net, params = _rand_net(widths, m=m, seed=7, bias_std=0.2)
    rng = np.random.default_rng(8)
    Pi = np.stack([rng.uniform(-1, 1, 40), rng.uniform(-1 if pde is POISSON else 0, 1, 40)], 1)
    Pb = rng.uniform(-1, 1, (12, 2))
    gb = rng.uniform(-0.5, 0.5, 12)
    lp, lb, grads = O.loss_grad(net, params, pde, Pi, Pb, gb)
    assert lp + lb == pytest.approx(O.loss(net, params, pde, Pi, Pb, gb), rel=1e-14)
    g_flat = O.flat_grad(grads)
    flat = HI.flatten_params(params).astype(np.float64)
    flat = O.flat_grad(params)
    h = 1e-30
    cs = np.empty_like(flat)
    for q in range(len(flat)):
        f = flat.astype(np.complex128)
        f[q] += 1j * h
        pr = HI.unflatten_params(f, widths, net.B)
        cs[q] = np.imag(O.loss(net, pr, pde, Pi, Pb, gb)) / h
    np.testing.assert_allclose(g_flat, cs, rtol=1e-10, atol=1e-13 * np.abs(cs).max())


def test_grad_central_fd_c2_shape():
    """30 random parameters, central FD with step 1e-6 max(1,|w|), rel < 1e-5."""
    w = HI.WORKLOADS["C2"]
    ps = HI.make_points(w).subset(20, 8)
    net, params = _rand_net(list(w.widths), seed=11, bias_std=0.1)
    bi = np.concatenate([ps.boundary, ps.initial])
    gbi = np.concatenate([ps.g_boundary, ps.g_initial])
    _, _, grads = O.loss_grad(net, params, BURGERS, ps.interior, bi, gbi)
    g = O.flat_grad(grads)
    flat = O.flat_grad(params)
    idx = np.random.default_rng(0).choice(len(flat), 30, replace=False)
    for q in idx:
        st = 1e-6 * max(1.0, abs(flat[q]))
        fp, fm = flat.copy(), flat.copy()
        fp[q] += st
        fm[q] -= st
        Lp = O.loss(net, HI.unflatten_params(fp, w.widths, w.B), BURGERS, ps.interior, bi, gbi)
        Lm = O.loss(net, HI.unflatten_params(fm, w.widths, w.B), BURGERS, ps.interior, bi, gbi)
        fd = (Lp - Lm) / (2 * st)
        assert abs(fd - g[q]) <= 1e-5 * max(abs(g[q]), 1e-3 * np.abs(g).max())


@pytest.mark.parametrize("key", ["C1", "C2"])
def test_grad_zero_weight_closed_form(key):
    """All W = 0, hidden biases non-zero, last bias beta: dL/db_last = 2 beta,
    dL/dW_last[0,i,n] = 2 beta v_n(b_prev,i), every other gradient 0."""
    w = HI.WORKLOADS[key]
    ps = HI.make_points(w)
    net = O.Net(w.widths, w.G, w.k, w.m)
    params = _zero_params(w.widths, w.B)
    rng = np.random.default_rng(1)
    for l in range(len(params) - 1):
        params[l] = (params[l][0], rng.uniform(-0.8, 0.8, len(params[l][1])))
    beta = 0.37
    params[-1] = (params[-1][0], np.array([beta]))
    pde = POISSON if w.pde == "poisson" else BURGERS
    bi = ps.boundary if ps.initial is None else np.concatenate([ps.boundary, ps.initial])
    gbi = ps.g_boundary if ps.initial is None else np.concatenate([ps.g_boundary, ps.g_initial])
    _, _, grads = O.loss_grad(net, params, pde, ps.interior, bi, gbi)
    bprev = params[-2][1]
    # L_bi = mean (beta - g)^2: derivative 2 mean(beta - g) = 2 beta - 2 mean(g)
    dbeta = 2 * beta - 2 * np.mean(gbi.astype(np.float64))
    assert grads[-1][1][0] == pytest.approx(dbeta, rel=1e-12)
    ref_W = dbeta * O.hr_basis(bprev[:, None], net.s, net.e, w.m, 0)
    np.testing.assert_allclose(grads[-1][0][0], ref_W, rtol=1e-12, atol=1e-15)
    for l in range(len(grads) - 1):
        assert np.abs(grads[l][0]).max() == 0.0 and np.abs(grads[l][1]).max() == 0.0


def test_grad_scales_with_loss():
    """scaling the loss scales every gradient (alpha and the boundary targets at 0)."""
    net, params = _rand_net([2, 4, 1], seed=2)
    P = np.random.default_rng(0).uniform(-1, 1, (30, 2))
    _, _, g1 = O.loss_grad(net, params, POISSON, P, P[:0], np.zeros(0))
    _, _, g10 = O.loss_grad(net, params, {**POISSON, "alpha": 0.5}, P, P[:0], np.zeros(0))
    np.testing.assert_allclose(O.flat_grad(g10), 10 * O.flat_grad(g1), rtol=1e-13, atol=1e-16)


def test_data_parallel_shard_sum():
    """Shard partial sums with global normalisers add up to the unsharded result (§8(e))."""
    w = HI.WORKLOADS["C2"]
    ps = HI.make_points(w).subset(10, 4)
    net, params = _rand_net(list(w.widths), seed=3)
    bi = np.concatenate([ps.boundary, ps.initial])
    gbi = np.concatenate([ps.g_boundary, ps.g_initial])
    lp, lb, g = O.loss_grad(net, params, BURGERS, ps.interior, bi, gbi)
    acc = np.zeros_like(O.flat_grad(g))
    lps = lbs = 0.0
    for r in range(3):
        sh = ps.shard(r, 3)
        sbi = np.concatenate([sh.boundary, sh.initial])
        sgbi = np.concatenate([sh.g_boundary, sh.g_initial])
        a, b, gg = O.loss_grad(net, params, BURGERS, sh.interior, sbi, sgbi,
                               n_int_global=len(ps.interior), n_bi_global=len(bi))
        lps += a
        lbs += b
        acc += O.flat_grad(gg)
    assert lps == pytest.approx(lp, rel=1e-12) and lbs == pytest.approx(lb, rel=1e-12)
    np.testing.assert_allclose(acc, O.flat_grad(g), rtol=1e-10, atol=1e-14)


# ---------------------------------------------------------------- Adam
def test_adam_one_step_closed_forms():
    th = np.array([0.5, -1.0, 2.0])
    z = np.zeros(3)
    # zero gradient at t=1 leaves the parameters unchanged
    t1, _, _ = O.adam_step(th, z, z, z, 1)
    np.testing.assert_array_equal(t1, th)
    # constant gradient, first step: delta = -lr g / (|g| + eps)
    g = np.array([0.3, -2.0, 1e-3])
    t1, m, v = O.adam_step(th, g, z, z, 1, lr=1e-3, eps=1e-8)
    np.testing.assert_allclose(t1 - th, -1e-3 * g / (np.abs(g) + 1e-8), rtol=1e-12)
    np.testing.assert_allclose(m, 0.1 * g, rtol=1e-15)
    np.testing.assert_allclose(v, 0.001 * g ** 2, rtol=1e-12)


# ---------------------------------------------------------------- residual pins on exact PDE solutions
def _burgers_travelling_wave(a, nu, c, A):
    """Exact travelling-wave solution of u_t + a u u_x - nu u_xx = 0 (Eq. 5, with the
    advection coefficient a): u = c - A tanh(a A (x - a c t) / (2 nu)).  Derived by integrating
    the travelling-wave ODE once (-s u + a u^2/2 - nu u' = const): matching the tanh^2 and tanh
    coefficients gives k = a A / (2 nu) and s = a c.  Returns sympy (x, t, u)."""
    x, t = sp.symbols("x t")
    u = c - A * sp.tanh(a * A * (x - a * c * t) / (2 * nu))
    return x, t, u


def _jet_of(u, x, t, P):
    f = sp.lambdify((x, t), [u, sp.diff(u, x), sp.diff(u, t), sp.diff(u, x, 2), sp.diff(u, t, 2)], "numpy")
    vals = [np.broadcast_to(np.asarray(v, np.float64), (len(P),)) for v in f(P[:, 0], P[:, 1])]
    uu, ux, ut, uxx, utt = vals
    return uu, np.stack([ux, ut], 1), np.stack([uxx, utt], 1)


@pytest.mark.parametrize("a,nu", [(1.0, 0.01 / np.pi), (0.25, 0.001 / 16), (0.7, 0.05)])
def test_burgers_residual_vanishes_on_exact_solution(a, nu):
    """burgers_residual (Eq. 5; Eq. 7, P:213 is a = 1/4, visc = nu/16) is zero on an exact
    solution of the same PDE while each of its three terms is O(1) there: a dropped term, a flipped
    sign, adv and visc swapped, or u_tt read for u_xx (u_tt = (a c)^2 u_xx here) all fail."""
    c, A = 0.3, 0.5
    x, t, u = _burgers_travelling_wave(sp.Rational(a).limit_denominator(10 ** 9), sp.Rational(nu).limit_denominator(10 ** 12), c, A)
    width = 2 * nu / (a * A)                              # the front's length scale
    rng = np.random.default_rng(5)
    tt = rng.uniform(0, 1, 64)
    xx = a * c * tt + rng.uniform(-2, 2, 64) * width       # points inside the front
    P = np.stack([xx, tt], 1)
    uu, du, d2u = _jet_of(u, x, t, P)
    r = O.burgers_residual(uu, du, d2u, a, nu)
    scale = np.abs(du[:, 1]) + np.abs(a * uu * du[:, 0]) + np.abs(nu * d2u[:, 0])
    assert np.median(np.abs(du[:, 1])) > 1e-2 * np.median(scale)   # every term is non-trivial
    assert np.median(np.abs(nu * d2u[:, 0])) > 1e-2 * np.median(scale)
    assert np.all(np.abs(r) <= 1e-9 * scale)
    # the wrong-reading variants do not vanish
    assert np.max(np.abs(du[:, 1] + a * uu * du[:, 0] + nu * d2u[:, 0]) / scale) > 0.1
    assert np.max(np.abs(du[:, 1] + a * uu * du[:, 0] - nu * d2u[:, 1]) / scale) > 0.1
    assert np.max(np.abs(du[:, 1] + nu * uu * du[:, 0] - a * d2u[:, 0]) / scale) > 0.1


def test_burgers_paper_change_of_variables():
    """y = (x + 5)/4 maps Eq. 5 with nu = 0.001 on [-5,5] to Eq. 7 (u_t + 1/4 u u_y -
    nu/16 u_yy = 0) on [0, 2.5].  An exact solution of Eq. 5, composed with x = 4y - 5, is zero under
    burgers_residual(adv=1/4, visc=nu/16) and not under (adv=1, visc=nu)."""
    nu = sp.Rational(1, 1000)
    x, t, u = _burgers_travelling_wave(1, nu, sp.Rational(3, 10), sp.Rational(1, 2))
    y = sp.symbols("y")
    w = u.subs(x, 4 * y - 5)
    rng = np.random.default_rng(6)
    tt = rng.uniform(0, 2.5, 64)
    yy = (0.3 * tt + 5 + rng.uniform(-2, 2, 64) * 2 * 0.001 / 0.5) / 4
    P = np.stack([yy, tt], 1)
    ww, dw, d2w = _jet_of(w, y, t, P)
    scale = np.abs(dw[:, 1]) + np.abs(0.25 * ww * dw[:, 0]) + np.abs(0.001 / 16 * d2w[:, 0])
    r = O.burgers_residual(ww, dw, d2w, 0.25, 0.001 / 16)
    assert np.all(np.abs(r) <= 1e-9 * scale)
    r_wrong = O.burgers_residual(ww, dw, d2w, 1.0, 0.001)
    assert np.max(np.abs(r_wrong) / scale) > 0.5


def test_poisson_forcing_3d():
    """BASELINE.json C5: f = -3 pi^2 prod_j sin(pi x_j).  At (1/2,1/2,1/2) f = -3 pi^2, so the residual
    of u == 0 is 3 pi^2; the exact solution prod_j sin(pi x_j) (laplacian -3 pi^2 prod sin) has zero
    residual; f vanishes on every face x_j = 0 of the inner cross."""
    half = np.array([[0.5, 0.5, 0.5]])
    assert O.poisson_forcing(half)[0] == pytest.approx(-3 * np.pi ** 2, rel=1e-15)
    assert O.poisson_residual(None, np.zeros((1, 3)), half)[0] == pytest.approx(3 * np.pi ** 2, rel=1e-15)
    assert O.poisson_forcing(np.array([[-0.5, 0.5, 0.5]]))[0] == pytest.approx(3 * np.pi ** 2, rel=1e-15)
    assert O.poisson_forcing(np.array([[0.3, 0.0, -0.7]]))[0] == 0.0
    P = np.random.default_rng(1).uniform(-1, 1, (200, 3))
    s = np.prod(np.sin(np.pi * P), axis=1)
    d2 = np.stack([-np.pi ** 2 * s] * 3, 1)
    assert np.abs(O.poisson_residual(None, d2, P)).max() < 1e-12
    # a 2-D forcing applied to 3-D points would carry 2 pi^2, not 3 pi^2
    assert abs(O.poisson_forcing(half)[0] + 2 * np.pi ** 2) > 1.0


def test_adam_constant_gradient_every_step():
    """with a constant gradient g, m_t = (1-b1^t) g and v_t = (1-b2^t) g^2, so the bias-corrected
    step is -lr g / (|g| + eps) at EVERY t (a bias correction frozen at t = 1, or missing, fails from t = 2)."""
    th0 = np.array([0.5, -1.0, 2.0, 0.0])
    g = np.array([0.3, -2.0, 1e-3, 5.0])
    th, m, v = th0.copy(), np.zeros(4), np.zeros(4)
    lr, eps = 1e-2, 1e-8
    for t in range(1, 6):
        prev = th
        th, m, v = O.adam_step(th, g, m, v, t, lr=lr, eps=eps)
        np.testing.assert_allclose(th - prev, -lr * g / (np.abs(g) + eps), rtol=1e-9)
        np.testing.assert_allclose(m, (1 - 0.9 ** t) * g, rtol=1e-12)
        np.testing.assert_allclose(v, (1 - 0.999 ** t) * g ** 2, rtol=1e-9)
    # a sign-alternating gradient: the first moment averages it, the step shrinks below lr
    th, m, v = th0.copy(), np.zeros(4), np.zeros(4)
    for t in range(1, 6):
        prev = th
        th, m, v = O.adam_step(th, (-1) ** t * g, m, v, t, lr=lr, eps=eps)
    assert np.all(np.abs(th - prev) < lr)
