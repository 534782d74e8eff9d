"""Float64 CPU oracle for the higher-order and mixed jets of SURVEY.md §8(f) row 3.

TEST INFRASTRUCTURE ONLY (same rule as hrkan_oracle.py): only `tests/`, `__graft_entry__.smoke()` and
bench.py's `cpu_baseline` / `--impl reference` legs may import this module; the product path never
does and shares no code with it.

What it computes (P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n):

* the Higher-order-ReLU basis v_{m,n}(x) = c_m [(e_n - x)(x - s_n)]^m (Eq. 2) and its x-derivatives
  of ANY order d, as the exact polynomial c_m p(x)^m expanded and differentiated d times with numpy's
  polynomial arithmetic (p = (e-x)(x-s) written in y = x - mid_n; no closed-form derivative formula), zero
  outside (s_n, e_n) (strict-interior reading 2);
* a univariate Taylor-mode jet of order R along one coordinate ("If a PDE equation possesses
  derivative terms of order higher than 4, for example, u_xxxxx, we can pick m to be larger, like 6"): each
  hidden value carries its truncated Taylor polynomial in eps along x, and a basis function is composed
  with it by substituting the polynomial into the basis's own Taylor expansion (truncated power-series
  composition, step by step); plus the first derivative along a second coordinate t;
* the full Hessian ("d2u: symmetric matrix of reals"; S:188 univariate chain rule): for z = phi(h),
  z_a = phi'(h) h_a and z_ab = phi''(h) h_a h_b + phi'(h) h_ab;
* residuals: the fifth-order Kawahara equation u_t + adv u u_x + disp3 u_xxx - disp5 u_xxxxx (a PDE with a
  u_xxxxx term) and an anisotropic second-order operator sum_{a<=b} K_ab u_ab - f (mixed terms);
* L = alpha L_pde + L_bi (Eq. 4 / Eq. 8 form) and dL/dtheta by torch.autograd in
  float64 on the CPU (a library reverse pass, independent of the CUDA path's hand-written one).

Pins: tests/test_oracle_jets.py (sympy-exact basis derivatives to order 8, continuity class C^{m-1}, exact
polynomial nets to fifth order / mixed second order, finite differences, the exact Kawahara solitary wave,
a manufactured anisotropic solution, agreement of the order-2 channels with hrkan_oracle.forward_jet,
finite-difference gradients).
"""
from __future__ import annotations

import math
from functools import lru_cache

import numpy as np
import torch
from numpy.polynomial import Polynomial

DT = torch.float64


# ----------------------------------------------------------------------------------------
# Basis of any derivative order (Eq. 2)
# ----------------------------------------------------------------------------------------
@lru_cache(maxsize=None)
def basis_poly_coeffs(w: float, m: int, d: int):
    """Coefficients (ascending powers of y = x - mid) of d^d/dx^d of c_m [(e - x)(x - s)]^m on a support of
    width w = e - s centred at mid: e - x = w/2 - y, x - s = w/2 + y.  Exact polynomial algebra."""
    p = Polynomial([w / 2.0, -1.0]) * Polynomial([w / 2.0, 1.0])      # (e - x)(x - s) in y
    c = (2.0 / w) ** (2 * m)                                          # c_m
    v = c * p ** m
    return tuple(v.deriv(d).coef) if d > 0 else tuple(v.coef)


def make_supports(G: int, k: int, lo: float, hi: float):
    """Same knots as hrkan_oracle.make_supports (DESIGN reading 1): s_n = lo + (n-k)h, e_n = s_n + (k+1)h."""
    h = (hi - lo) / G
    n = np.arange(G + k, dtype=np.float64)
    s = lo + (n - k) * h
    return s, s + (k + 1) * h


def basis(x: torch.Tensor, s: np.ndarray, e: np.ndarray, m: int, d: int) -> torch.Tensor:
    """v^{(d)}_{m,n}(x) for every n: x[...] -> [..., B].  Horner in y = x - mid_n; exactly 0 outside (s_n, e_n)."""
    s_t = torch.as_tensor(s, dtype=DT)
    e_t = torch.as_tensor(e, dtype=DT)
    w = float(e[0] - s[0])
    coef = basis_poly_coeffs(w, m, d)
    y = x[..., None] - 0.5 * (s_t + e_t)
    acc = torch.zeros_like(y)
    for a in reversed(coef):
        acc = acc * y + a
    inside = (x[..., None] > s_t) & (x[..., None] < e_t)
    return torch.where(inside, acc, torch.zeros_like(acc))


class Net:
    def __init__(self, widths, G, k, m, lo=-1.0, hi=1.0):
        self.widths = list(widths)
        self.G, self.k, self.m, self.lo, self.hi = G, k, m, lo, hi
        self.B = G + k
        self.s, self.e = make_supports(G, k, lo, hi)

    def phi(self, x, d):
        return basis(x, self.s, self.e, self.m, d)


def params_to_torch(params, requires_grad=False):
    out = []
    for W, b in params:
        Wt = torch.tensor(np.asarray(W, np.float64), dtype=DT, requires_grad=requires_grad)
        bt = torch.tensor(np.asarray(b, np.float64), dtype=DT, requires_grad=requires_grad)
        out.append((Wt, bt))
    return out


# ----------------------------------------------------------------------------------------
# Taylor-mode jet along x (order R) + first derivative along t
# ----------------------------------------------------------------------------------------
def _series_mul(a, b, R):
    """Truncated product of two power series in eps: coefficient tensors [..., R+1]."""
    out = torch.zeros_like(a)
    for i in range(R + 1):
        for j in range(R + 1 - i):
            out[..., i + j] = out[..., i + j] + a[..., i] * b[..., j]
    return out


def compose_taylor(net: Net, h, R: int):
    """phi_n(h(eps)) as a power series in eps, for every basis n.

    h[..., R+1]: Taylor coefficients of the input (h_0 + h_1 eps + ... ; h_r = d^r h/dx^r / r!).
    phi(h_0 + delta) = sum_{k=0}^{R} phi^{(k)}(h_0)/k! delta^k with delta = sum_{r>=1} h_r eps^r, every
    product truncated at eps^R.  Returns [..., B, R+1] series coefficients."""
    h0 = h[..., 0]
    delta = h.clone()
    delta[..., 0] = 0.0
    delta = delta[..., None, :]                                  # [..., 1, R+1] broadcast over n
    out = None
    power = torch.zeros(h.shape[:-1] + (1, R + 1), dtype=DT)
    power[..., 0] = 1.0                                          # delta^0
    for k in range(R + 1):
        term = net.phi(h0, k)[..., None] / math.factorial(k) * power   # [..., B, R+1]
        out = term if out is None else out + term
        power = _series_mul(power.expand_as(term), delta.expand_as(term), R)
    return out


def forward_taylor(net: Net, params_t, pts, R: int, xdir: int = 0, tdir: int = 1):
    """u and its derivatives d^r u/dx^r (r = 0..R) along coordinate xdir, plus du/dt along tdir.

    Returns (ux[P, R+1] derivatives, ut[P]).  Input jet of layer 0: x_i = xi_i; the x-series of input i is
    xi_i + [i == xdir] eps; the t-derivative of input i is [i == tdir]."""
    pts = torch.as_tensor(np.asarray(pts, np.float64), dtype=DT)
    P, D = pts.shape
    ser = torch.zeros(P, D, R + 1, dtype=DT)
    ser[..., 0] = pts
    if R >= 1:
        ser[:, xdir, 1] = 1.0
    ht = torch.zeros(P, D, dtype=DT)
    if tdir is not None and tdir < D:
        ht[:, tdir] = 1.0
    for W, b in params_t:
        comp = compose_taylor(net, ser, R)                       # [P, I, B, R+1]
        dphi = net.phi(ser[..., 0], 1)                           # [P, I, B]
        ser = torch.einsum("jin,pinr->pjr", W, comp)
        ser = ser + torch.cat([b[None, :, None], torch.zeros(1, len(b), R, dtype=DT)], dim=2)
        ht = torch.einsum("jin,pin->pj", W, dphi * ht[..., None])
    fact = torch.tensor([math.factorial(r) for r in range(R + 1)], dtype=DT)
    return ser[:, 0, :] * fact, ht[:, 0]


# ----------------------------------------------------------------------------------------
# Full Hessian jet
# ----------------------------------------------------------------------------------------
def forward_hessian(net: Net, params_t, pts):
    """u[P], grad[P, D], hess[P, D, D] (symmetric) by the second-order univariate chain rule per edge."""
    x = torch.as_tensor(np.asarray(pts, np.float64), dtype=DT)
    P, D = x.shape
    g = torch.eye(D, dtype=DT).expand(P, D, D).clone()          # g[p, i, a] = d x_i / d xi_a
    H = torch.zeros(P, D, D, D, dtype=DT)                       # H[p, i, a, b]
    for W, b in params_t:
        f0, f1, f2 = net.phi(x, 0), net.phi(x, 1), net.phi(x, 2)    # [P, I, B]
        y = torch.einsum("jin,pin->pj", W, f0) + b
        gy = torch.einsum("jin,pin,pia->pja", W, f1, g)
        Hy = (torch.einsum("jin,pin,pia,pib->pjab", W, f2, g, g)
              + torch.einsum("jin,pin,piab->pjab", W, f1, H))
        x, g, H = y, gy, Hy
    return x[:, 0], g[:, 0], H[:, 0]


def pair_index(D: int):
    """Upper-triangle (a <= b) pairs in row-major order: D=2 -> (0,0),(0,1),(1,1)."""
    return [(a, b) for a in range(D) for b in range(a, D)]


# ----------------------------------------------------------------------------------------
# Residuals and loss
# ----------------------------------------------------------------------------------------
def kawahara_residual(u, ux, ut, adv, disp3, disp5):
    """r = u_t + adv u u_x + disp3 u_xxx - disp5 u_xxxxx  (fifth-order KdV / Kawahara form; ux[:, r] = d^r u/dx^r)."""
    return ut + adv * u * ux[:, 1] + disp3 * ux[:, 3] - disp5 * ux[:, 5]


def aniso_residual(hess, K, forcing):
    """r = sum_{a<=b} K[(a,b)] u_ab - f, K over the upper-triangle pairs (pair_index)."""
    D = hess.shape[1]
    r = -torch.as_tensor(np.asarray(forcing, np.float64), dtype=DT)
    for q, (a, b) in enumerate(pair_index(D)):
        r = r + float(K[q]) * hess[:, a, b]
    return r


def value(net: Net, params_t, pts):
    x = torch.as_tensor(np.asarray(pts, np.float64), dtype=DT)
    for W, b in params_t:
        x = torch.einsum("jin,pin->pj", W, net.phi(x, 0)) + b
    return x[:, 0]


def loss_parts(net: Net, params_t, pde: dict, pts_int, pts_bi, g_bi, n_int_global=None, n_bi_global=None,
               forcing=None):
    """(alpha L_pde part, L_bi part) as torch scalars; pooled boundary/initial normaliser."""
    n_int = len(pts_int) if n_int_global is None else n_int_global
    n_bi = len(pts_bi) if n_bi_global is None else n_bi_global
    lp = torch.zeros((), dtype=DT)
    lb = torch.zeros((), dtype=DT)
    if len(pts_int):
        if pde["kind"] == "kawahara":
            ux, ut = forward_taylor(net, params_t, pts_int, 5)
            r = kawahara_residual(ux[:, 0], ux, ut, pde["adv"], pde["disp3"], pde["disp5"])
        elif pde["kind"] == "aniso":
            _, _, H = forward_hessian(net, params_t, pts_int)
            r = aniso_residual(H, pde["K"], forcing)
        else:
            raise ValueError(pde["kind"])
        lp = pde["alpha"] * (r * r).sum() / n_int
    if len(pts_bi):
        eb = value(net, params_t, pts_bi) - torch.as_tensor(np.asarray(g_bi, np.float64), dtype=DT)
        lb = (eb * eb).sum() / n_bi
    return lp, lb


def loss_grad(net: Net, params, pde: dict, pts_int, pts_bi, g_bi, n_int_global=None, n_bi_global=None,
              forcing=None):
    """(alpha L_pde part, L_bi part, [(dW_l, db_l)]) as float64 numpy; gradients by torch.autograd."""
    pt = params_to_torch(params, requires_grad=True)
    lp, lb = loss_parts(net, pt, pde, pts_int, pts_bi, g_bi, n_int_global, n_bi_global, forcing)
    L = lp + lb
    flat = [t for pair in pt for t in pair]
    if not L.requires_grad:                      # no points at all: L = 0, every gradient 0
        return float(lp), float(lb), [(np.zeros_like(np.asarray(W, np.float64)), np.zeros_like(np.asarray(b, np.float64)))
                                      for W, b in params]
    grads = torch.autograd.grad(L, flat, allow_unused=True)
    grads = [torch.zeros_like(t) if g is None else g for t, g in zip(flat, grads)]
    out = [(grads[2 * l].numpy(), grads[2 * l + 1].numpy()) for l in range(len(pt))]
    return float(lp.detach()), float(lb.detach()), out


def flat_grad(grads) -> np.ndarray:
    """Flat layout of include/hrkan.h: per layer W[O][I][B] then b[O]."""
    return np.concatenate([np.concatenate([np.ravel(W), np.ravel(b)]) for W, b in grads])
