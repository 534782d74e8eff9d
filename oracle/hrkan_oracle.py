"""Float64 CPU oracle for the HRKAN physics-informed loss + gradient step.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the `cpu_baseline` /
`--impl reference` legs of `bench.py` may import this module.  The product path
(`paper_2409_14248_b200/`) never imports it and shares no code with it.

Plain, slow, obviously correct numpy in float64 (dtype-generic so that complex-step
differentiation works: every branch tests the REAL part of its argument).  Each function
cites the passage it follows: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n,
SURVEY §8(c) = the readings adopted where the paper is silent (listed in DESIGN.md).

Pins (tests/test_oracle_*.py, `-m "not gpu"`): basis normalisation / support / continuity
class / quadrature / ReLU^2 special case / worked value 0.31640625 / FD derivatives; jets
vs sympy-exact polynomial nets and FD; loss vs zero-weight closed forms; gradient vs
complex-step and FD; Adam one-step closed form.  Nothing here is "parity unpinned".
"""
from __future__ import annotations

import numpy as np


def _f(a):
    """float64 (or complex128 for complex-step checks) view of an input array."""
    a = np.asarray(a)
    return a if np.iscomplexobj(a) else a.astype(np.float64)


# ----------------------------------------------------------------------------------------
# Basis  (Sec. 3 Eq. 2)
# ----------------------------------------------------------------------------------------
def make_supports(G: int, k: int, lo: float, hi: float):
    """Supports "the same as the B-splines"; uniform extended knots
    t_j = lo + j h, h = (hi-lo)/G, support n = [t_{n-k}, t_{n+1}].
    Returns (s[B], e[B]) float64 arrays, B = G + k (n = g + k basis functions)."""
    if G < 1 or k < 1 or not lo < hi:
        raise ValueError("invalid basis config")
    h = (hi - lo) / G
    n = np.arange(G + k, dtype=np.float64)
    s = lo + (n - k) * h
    e = s + (k + 1) * h
    return s, e


def c_m(s, e, m: int):
    """Normalisation constant c_m = (2/(e_i - s_i))^{2m}."""
    return (2.0 / (e - s)) ** (2 * m)


def hr_basis(x, s, e, m: int, d: int = 0):
    """d-th derivative (d = 0..3) of v_{m,i}(x) = ReLU(e_i-x)^m ReLU(x-s_i)^m c_m  (Eq. 2).

    Written in the literal product form with p = (e-x)(x-s), p' = e+s-2x, p'' = -2:
      v   = c p^m
      v'  = c m p^{m-1} p'
      v'' = c m p^{m-2} [ (m-1) p'^2 - 2 p ]
      v'''= c m (m-1) p' [ (m-2) p^{m-3} p'^2 - 6 p^{m-2} ]
    valid strictly inside (s, e); every derivative is exactly 0 outside, ReLU(0) = 0
    (SURVEY §8(c) reading 2: strict-interior convention at the knots).
    Broadcasts x against (s, e)."""
    x = np.asarray(x)
    s = np.asarray(s, dtype=np.float64)
    e = np.asarray(e, dtype=np.float64)
    c = c_m(s, e, m)
    p = (e - x) * (x - s)
    dp = e + s - 2.0 * x
    if d == 0:
        v = c * p ** m
    elif d == 1:
        v = c * m * p ** (m - 1) * dp
    elif d == 2:
        v = c * m * p ** (m - 2) * ((m - 1) * dp ** 2 - 2.0 * p)
    elif d == 3:
        first = (m - 2) * p ** (m - 3) * dp ** 2 if m >= 3 else 0.0 * p
        v = c * m * (m - 1) * dp * (first - 6.0 * p ** (m - 2))
    else:
        raise ValueError("d must be 0..3")
    xr = np.real(x)
    inside = (xr > s) & (xr < e)
    return np.where(inside, v, 0.0 * v)


def relu2_basis(x, s, e):
    """'Square of ReLU' r_i(x) = [ReLU(e_i-x) ReLU(x-s_i)]^2 c, c = 16/(e_i-s_i)^4 (Eq. 1).
    Independent formula used only to pin hr_basis at m = 2."""
    x = np.asarray(x)
    c = 16.0 / (e - s) ** 4
    xr = np.real(x)
    inside = (xr > s) & (xr < e)
    return np.where(inside, ((e - x) * (x - s)) ** 2 * c, 0.0 * x)


# ----------------------------------------------------------------------------------------
# Network forward jet ("matrix operation")
# ----------------------------------------------------------------------------------------
class Net:
    """widths [D, ..., 1], basis (G, k, m, lo, hi); params = list of (W[O,I,B], b[O]).
    Bias on the value channel only (SURVEY §8(c) reading 3; BASELINE.json "bias gradient")."""

    def __init__(self, widths, G, k, m, lo=-1.0, hi=1.0):
        self.widths = list(widths)
        self.G, self.k, self.m = G, k, m
        self.lo, self.hi = lo, hi
        self.s, self.e = make_supports(G, k, lo, hi)
        self.B = G + k

    def features(self, x, d):
        """A^{(d)}[p,i,n] = v^{(d)}_{m,n}(x[p,i])."""
        return hr_basis(x[..., None], self.s, self.e, self.m, d)


def layer_forward(net: Net, W, b, x, dx, ddx):
    """One KAN layer applied to a diagonal second-order jet.

    x[p,i], dx[p,i,a] = dx_i/dxi_a, ddx[p,i,a] = d^2 x_i/dxi_a^2.  With phi = basis(x):
      A0[p,i,n]   = phi_n(x_i)
      A1[p,a,i,n] = phi'_n(x_i) dx_{i,a}
      A2[p,a,i,n] = phi''_n(x_i) dx_{i,a}^2 + phi'_n(x_i) ddx_{i,a}   (univariate chain rule)
      y_j = b_j + sum_{i,n} W[j,i,n] A0,  y'_{j,a} = sum W A1,  y''_{j,a} = sum W A2."""
    f0 = net.features(x, 0)
    f1 = net.features(x, 1)
    f2 = net.features(x, 2)
    A0 = f0
    A1 = f1[:, None, :, :] * np.transpose(dx, (0, 2, 1))[..., None]
    A2 = (f2[:, None, :, :] * np.transpose(dx, (0, 2, 1))[..., None] ** 2
          + f1[:, None, :, :] * np.transpose(ddx, (0, 2, 1))[..., None])
    y = np.einsum("jin,pin->pj", W, A0) + b[None, :]
    dy = np.einsum("jin,pain->pja", W, A1)
    ddy = np.einsum("jin,pain->pja", W, A2)
    return y, dy, ddy


def forward_jet(net: Net, params, pts, return_saved=False):
    """u, du[:, a], d2u[:, a] (diagonal) at points pts[P, D].  Layer-0 input jet:
    x_i = xi_i, dx_{i,a} = delta_ia, ddx = 0.  No clamping of hidden
    values outside [lo, hi]."""
    pts = np.asarray(pts)
    P, D = pts.shape
    x = pts.astype(np.result_type(pts.dtype, np.float64))
    dx = np.broadcast_to(np.eye(D)[None], (P, D, D)).astype(x.dtype)
    ddx = np.zeros((P, D, D), dtype=x.dtype)
    saved = []
    for (W, b) in params:
        saved.append((x, dx, ddx))
        x, dx, ddx = layer_forward(net, _f(W), _f(b), x, dx, ddx)
    u, du, d2u = x[:, 0], dx[:, 0, :], ddx[:, 0, :]
    if return_saved:
        return u, du, d2u, saved
    return u, du, d2u


def forward_value(net: Net, params, pts):
    """Value-only forward (boundary / initial points)."""
    x = np.asarray(pts).astype(np.result_type(np.asarray(pts).dtype, np.float64))
    for (W, b) in params:
        x = np.einsum("jin,pin->pj", _f(W), net.features(x, 0)) + _f(b)
    return x[:, 0]


# ----------------------------------------------------------------------------------------
# PDE residuals and loss  (Eq. 3-4;  P:195-238 Eq. 5-8;  BASELINE.json forms)
# ----------------------------------------------------------------------------------------
def poisson_forcing(pts):
    """f = -D pi^2 prod_a sin(pi xi_a)   (Eq. 3, for D=2; BASELINE.json C5 for D=3)."""
    pts = np.asarray(pts, dtype=np.float64)
    D = pts.shape[1]
    return -D * np.pi ** 2 * np.prod(np.sin(np.pi * pts), axis=1)


def poisson_residual(du, d2u, pts, forcing=None):
    """r = sum_a u_aa - f  (Eq. 3: laplacian u = f; L_pde summand of Eq. 4)."""
    f = poisson_forcing(pts) if forcing is None else np.asarray(forcing, np.float64)
    return d2u.sum(axis=1) - f


def burgers_residual(u, du, d2u, adv, visc):
    """r = u_t + adv u u_x - visc u_xx, coordinates (x, t)  (Eq. 5 P:197 with adv=1, visc=nu;
    the paper's transformed Eq. 7 P:213 is adv=1/4, visc=nu/16)."""
    return du[:, 1] + adv * u * du[:, 0] - visc * d2u[:, 0]


def loss_parts(net, params, pde, pts_int, pts_bi, g_bi, n_int_global=None, n_bi_global=None,
               forcing=None):
    """L = alpha L_pde + L_bi with L_pde = (1/N_int) sum r^2, L_bi = (1/N_bi) sum (u - g)^2 over
    the POOLED boundary (+ initial) set.  With global normalisers the
    parts of the shards of a data-parallel split add up to the unsharded parts.
    Returns (alpha*L_pde part, L_bi part)."""
    n_int_global = len(pts_int) if n_int_global is None else n_int_global
    n_bi_global = len(pts_bi) if n_bi_global is None else n_bi_global
    u, du, d2u = forward_jet(net, params, pts_int)
    r = _residual(pde, u, du, d2u, pts_int, forcing)
    ub = forward_value(net, params, pts_bi)
    lp = pde["alpha"] * np.sum(r ** 2) / n_int_global if len(pts_int) else 0.0
    lb = np.sum((ub - np.asarray(g_bi, np.float64)) ** 2) / n_bi_global if len(pts_bi) else 0.0
    return lp, lb


def loss(net, params, pde, pts_int, pts_bi, g_bi, **kw):
    lp, lb = loss_parts(net, params, pde, pts_int, pts_bi, g_bi, **kw)
    return lp + lb


def _residual(pde, u, du, d2u, pts, forcing):
    if pde["kind"] == "poisson":
        return poisson_residual(du, d2u, pts, forcing)
    return burgers_residual(u, du, d2u, pde["adv"], pde["visc"])


# ----------------------------------------------------------------------------------------
# Reverse pass  (the jet chain needs phi''' -- S:247)
# ----------------------------------------------------------------------------------------
def layer_backward(net: Net, W, x, dx, ddx, gy, gdy, gddy):
    """Adjoints of one layer.  gy[p,j], gdy[p,j,a], gddy[p,j,a] = dL/d(y, y', y'').
      dW[j,i,n] = sum_p gy A0 + sum_{p,a} gdy A1 + gddy A2,   db_j = sum_p gy
      Abar^c[p,(a),i,n] = sum_j g^c_j W[j,i,n]
      xbar      = sum_n [Abar0 phi' + sum_a Abar1_a phi'' dx_a + sum_a Abar2_a (phi''' dx_a^2 + phi'' ddx_a)]
      dxbar_a   = sum_n [Abar1_a phi' + 2 Abar2_a phi'' dx_a]
      ddxbar_a  = sum_n  Abar2_a phi'
    Returns (dW, db, xbar, dxbar, ddxbar)."""
    f0 = net.features(x, 0)
    f1 = net.features(x, 1)
    f2 = net.features(x, 2)
    f3 = net.features(x, 3)
    dxT = np.transpose(dx, (0, 2, 1))[..., None]     # [p,a,i,1]
    ddxT = np.transpose(ddx, (0, 2, 1))[..., None]
    A0 = f0
    A1 = f1[:, None] * dxT
    A2 = f2[:, None] * dxT ** 2 + f1[:, None] * ddxT
    dW = (np.einsum("pj,pin->jin", gy, A0) + np.einsum("pja,pain->jin", gdy, A1)
          + np.einsum("pja,pain->jin", gddy, A2))
    db = gy.sum(axis=0)
    Ab0 = np.einsum("pj,jin->pin", gy, W)
    Ab1 = np.einsum("pja,jin->pain", gdy, W)
    Ab2 = np.einsum("pja,jin->pain", gddy, W)
    xbar = (np.sum(Ab0 * f1, axis=2)
            + np.sum(Ab1 * f2[:, None] * dxT, axis=(1, 3))
            + np.sum(Ab2 * (f3[:, None] * dxT ** 2 + f2[:, None] * ddxT), axis=(1, 3)))
    dxbar = np.sum(Ab1 * f1[:, None] + 2.0 * Ab2 * f2[:, None] * dxT, axis=3)   # [p,a,i]
    ddxbar = np.sum(Ab2 * f1[:, None], axis=3)
    return dW, db, xbar, np.transpose(dxbar, (0, 2, 1)), np.transpose(ddxbar, (0, 2, 1))


def loss_grad(net, params, pde, pts_int, pts_bi, g_bi, n_int_global=None, n_bi_global=None,
              forcing=None):
    """(alpha L_pde part, L_bi part, [(dW_l, db_l)]) by the hand-written reverse pass.

    Seeds at the last layer, g = 2 alpha r / N_int:
      Poisson interior: dL/du_aa = g for every a
      Burgers interior: dL/du = g adv u_x, dL/du_x = g adv u, dL/du_t = g, dL/du_xx = -g visc
      boundary/initial: dL/du = 2 (u - g_bi) / N_bi."""
    pts_int = _f(pts_int).reshape(-1, net.widths[0])
    pts_bi = _f(pts_bi).reshape(-1, net.widths[0])
    n_int_global = len(pts_int) if n_int_global is None else n_int_global
    n_bi_global = len(pts_bi) if n_bi_global is None else n_bi_global
    alpha = pde["alpha"]
    L = len(params)
    grads = [[0.0, 0.0] for _ in params]
    lp = lb = 0.0
    # interior: full jet
    if len(pts_int):
        u, du, d2u, saved = forward_jet(net, params, pts_int, return_saved=True)
        r = _residual(pde, u, du, d2u, pts_int, forcing)
        lp = alpha * np.sum(r ** 2) / n_int_global
        g = 2.0 * alpha * r / n_int_global
        P, D = pts_int.shape
        gy = np.zeros((P, 1))
        gdy = np.zeros((P, 1, D))
        gddy = np.zeros((P, 1, D))
        if pde["kind"] == "poisson":
            gddy[:, 0, :] = g[:, None]
        else:
            gy[:, 0] = g * pde["adv"] * du[:, 0]
            gdy[:, 0, 0] = g * pde["adv"] * u
            gdy[:, 0, 1] = g
            gddy[:, 0, 0] = -g * pde["visc"]
        for l in range(L - 1, -1, -1):
            x, dx, ddx = saved[l]
            dW, db, xb, dxb, ddxb = layer_backward(net, _f(params[l][0]),
                                                   x, dx, ddx, gy, gdy, gddy)
            grads[l][0] += dW
            grads[l][1] += db
            gy, gdy, gddy = xb, dxb, ddxb
    # boundary + initial: value-only jet (C = 1)
    if len(pts_bi):
        P, D = pts_bi.shape
        xs = []
        x = pts_bi
        for (W, b) in params:
            xs.append(x)
            x = np.einsum("jin,pin->pj", _f(W), net.features(x, 0)) + _f(b)
        ub = x[:, 0]
        e = ub - np.asarray(g_bi, np.float64)
        lb = np.sum(e ** 2) / n_bi_global
        gy = (2.0 * e / n_bi_global)[:, None]
        for l in range(L - 1, -1, -1):
            xin = xs[l]
            I = xin.shape[1]
            zero = np.zeros((P, I, 1))
            dW, db, xb, _, _ = layer_backward(net, _f(params[l][0]), xin, zero, zero,
                                              gy, np.zeros((P, gy.shape[1], 1)), np.zeros((P, gy.shape[1], 1)))
            grads[l][0] += dW
            grads[l][1] += db
            gy = xb
    return lp, lb, [(g[0], g[1]) for g in grads]


# ----------------------------------------------------------------------------------------
# Adam  ("Adam optimizer"; hyper-parameters unstated -> S:280 defaults)
# ----------------------------------------------------------------------------------------
def adam_step(theta, grad, m, v, t, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8):
    """Standard bias-corrected Adam.  t is the step index AFTER increment (>= 1).
    Returns (theta, m, v)."""
    m = beta1 * m + (1.0 - beta1) * grad
    v = beta2 * v + (1.0 - beta2) * grad ** 2
    mhat = m / (1.0 - beta1 ** t)
    vhat = v / (1.0 - beta2 ** t)
    return theta - lr * mhat / (np.sqrt(vhat) + eps), m, v


def flat_grad(grads) -> np.ndarray:
    """Flat layout of include/hrkan.h: per layer W[O][I][B] then b[O]."""
    return np.concatenate([np.concatenate([np.ravel(W), np.ravel(b)]) for W, b in grads])
