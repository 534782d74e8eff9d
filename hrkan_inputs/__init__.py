"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the HRKAN method (no basis, no jet, no residual, no loss,
no gradient).  It only draws collocation points, boundary/initial targets and random
parameters, so that the float64 oracle (`oracle/`) and the CUDA path
(`paper_2409_14248_b200/`) can be fed identical inputs without sharing code.

Workload recipe (BASELINE.json `configs`):

* C1  2D Poisson [2,5,1], G=5,k=3,m=4: 32x32 cell-centred interior grid on (-1,1)^2,
      4 edges x linspace(-1,1,32) boundary points, g=0.  Shape of the paper's
      960 + 4x30 Poisson set (Sec. 4.1).
* C2  Burgers [2,5,5,1], G=5,k=3,m=4, nu=0.01/pi: 10 000 iid U([-1,1]x[0,1]) interior
      points (the paper's N_pde = 10000), 256 initial points
      x=linspace(-1,1,256), t=0, g=-sin(pi x); 128+128 boundary points at x=-1 / x=+1,
      t=linspace(0,1,128), g=0.
* C3  2D Poisson [2,64,64,1], G=10: 2^20 iid U((-1,1)^2) + 4x1024 edge points.
* C4  Burgers [2,128,128,128,1], G=8, m in {2,3,4}: 2^22 iid interior, 2^14 initial
      (linspace x), 2^14 boundary (2^13 per side, linspace t).
* C5  3D Poisson [3,256,256,1], G=16: 2^24 iid U((-1,1)^3), 2^16 boundary points,
      face = q mod 6, uniform on that face, g=0.

Points are drawn in float64 with numpy PCG64 and rounded to float32; both sides consume
those float32 values (the oracle upcasts them).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np

POINT_SEED = 0
PARAM_SEED = 1


@dataclass(frozen=True)
class Workload:
    key: str
    name: str
    pde: str                    # "poisson" | "burgers"
    widths: tuple
    G: int
    k: int
    m: int
    n_int: int
    n_bnd: int
    n_ic: int
    lo: float = -1.0
    hi: float = 1.0
    alpha: float = 0.05         # PAPER.md:142 / :239
    adv: float = 1.0            # Burgers r = u_t + adv*u*u_x - visc*u_xx (BASELINE.json form)
    visc: float = 0.01 / math.pi
    disp3: float = 0.0          # Kawahara r = u_t + adv u u_x + disp3 u_xxx - disp5 u_xxxxx
    disp5: float = 0.0
    aniso: tuple = ()           # anisotropic r = sum_{a<=b} aniso[q] u_ab - f (upper triangle, row-major)

    @property
    def D(self) -> int:
        return self.widths[0]

    @property
    def B(self) -> int:
        return self.G + self.k

    @property
    def n_points(self) -> int:
        return self.n_int + self.n_bnd + self.n_ic

    def num_params(self) -> int:
        w = self.widths
        return sum(w[l + 1] * w[l] * self.B + w[l + 1] for l in range(len(w) - 1))

    def with_m(self, m: int) -> "Workload":
        return Workload(**{**self.__dict__, "m": m, "key": f"{self.key.split('_')[0]}_m{m}"})


WORKLOADS: Dict[str, Workload] = {
    "C1": Workload("C1", "poisson2d_[2,5,1]_G5_k3_m4", "poisson", (2, 5, 1), 5, 3, 4, 1024, 128, 0),
    "C2": Workload("C2", "burgers_[2,5,5,1]_G5_k3_m4", "burgers", (2, 5, 5, 1), 5, 3, 4, 10000, 256, 256),
    "C3": Workload("C3", "poisson2d_[2,64,64,1]_G10_k3_m4", "poisson", (2, 64, 64, 1), 10, 3, 4,
                   1 << 20, 4096, 0),
    "C4": Workload("C4", "burgers_[2,128,128,128,1]_G8_k3_m4", "burgers", (2, 128, 128, 128, 1), 8, 3, 4,
                   1 << 22, 1 << 14, 1 << 14),
    "C5": Workload("C5", "poisson3d_[3,256,256,1]_G16_k3_m4", "poisson", (3, 256, 256, 1), 16, 3, 4,
                   1 << 24, 1 << 16, 0),
    # the paper's own experiments (parity cases, not bench lines): Sec. 4.1 Poisson (PAPER.md:110-142,
    # [2,2,1], g=5, 960 random interior + 4 x 30 equally spaced boundary points) and Sec. 4.2 transformed
    # Burgers (Eq. 7: adv = 1/4, visc = nu/16, nu = 0.001, (y,t) in [0,2.5]^2,
    # [2,3,3,3,1], g=7, 10000 interior + 100 + 100 boundary + 100 initial points, u(y,0) = 1/cosh(4y-5))
    "PP": Workload("PP", "paper_poisson_[2,2,1]_G5_k3_m4", "poisson", (2, 2, 1), 5, 3, 4, 960, 120, 0),
    "PB": Workload("PB", "paper_burgers_[2,3,3,3,1]_G7_k3_m4", "burgers", (2, 3, 3, 3, 1), 7, 3, 4, 10000, 200, 100,
                   lo=0.0, hi=2.5, adv=0.25, visc=0.001 / 16),
    # SURVEY §8(f) row 3 (higher-order and mixed jets; PAPER.md:102 picks m = 6 for a u_xxxxx term):
    #   K*: Kawahara u_t + u u_x + 0.01 u_xxx - 1e-4 u_xxxxx = 0 on [-1,1] x [0,1], exact solitary-wave
    #       initial and boundary values (Taylor-5 jet); A*: anisotropic operator with mixed second
    #       derivatives, manufactured u* = prod sin(pi x_a), forcing from u*, u = 0 on the boundary.
    "K1": Workload("K1", "kawahara_[2,16,16,1]_G8_k3_m6", "kawahara", (2, 16, 16, 1), 8, 3, 6, 4096, 256, 256,
                   adv=1.0, visc=0.0, disp3=0.01, disp5=1e-4),
    "K6": Workload("K6", "kawahara_[2,64,64,1]_G10_k3_m6", "kawahara", (2, 64, 64, 1), 10, 3, 6, 1 << 20, 1 << 12,
                   1 << 12, adv=1.0, visc=0.0, disp3=0.01, disp5=1e-4),
    "A2": Workload("A2", "aniso2d_[2,32,32,1]_G8_k3_m4", "aniso", (2, 32, 32, 1), 8, 3, 4, 4096, 256, 0,
                   aniso=(1.0, 0.6, 0.5)),
    "A3": Workload("A3", "aniso3d_[3,32,32,1]_G8_k3_m6", "aniso", (3, 32, 32, 1), 8, 3, 6, 4096, 384, 0,
                   aniso=(1.0, 0.4, 0.2, 0.8, 0.3, 0.6)),
}


@dataclass
class PointSet:
    interior: np.ndarray                  # [Ni, D] float32
    boundary: np.ndarray                  # [Nb, D] float32
    g_boundary: np.ndarray                # [Nb]    float32
    initial: Optional[np.ndarray] = None  # [N0, D] float32 (Burgers)
    g_initial: Optional[np.ndarray] = None
    forcing: Optional[np.ndarray] = None  # [Ni] float32 (anisotropic operator: f of the manufactured solution)

    @property
    def n_bi(self) -> int:
        return len(self.boundary) + (0 if self.initial is None else len(self.initial))

    def subset(self, s_int: int, s_bi: int) -> "PointSet":
        """Every s-th point of each set (strided, so every edge/face stays represented)."""
        return PointSet(
            self.interior[::s_int].copy(), self.boundary[::s_bi].copy(), self.g_boundary[::s_bi].copy(),
            None if self.initial is None else self.initial[::s_bi].copy(),
            None if self.g_initial is None else self.g_initial[::s_bi].copy(),
            None if self.forcing is None else self.forcing[::s_int].copy())

    def shard(self, rank: int, world: int) -> "PointSet":
        """Contiguous equal blocks per rank (the DP partition of SURVEY.md §8(e))."""
        def blk(a):
            if a is None:
                return None
            n = len(a)
            lo = (n * rank) // world
            hi = (n * (rank + 1)) // world
            return a[lo:hi]
        return PointSet(blk(self.interior), blk(self.boundary), blk(self.g_boundary),
                        blk(self.initial), blk(self.g_initial), blk(self.forcing))


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64).astype(np.float32))


def _edges_2d(n_per_edge: int) -> np.ndarray:
    t = np.linspace(-1.0, 1.0, n_per_edge)
    one = np.ones_like(t)
    return np.concatenate([np.stack([-one, t], 1), np.stack([one, t], 1),
                           np.stack([t, -one], 1), np.stack([t, one], 1)], 0)


def kawahara_wave(x, t, w: Workload, x0: float = -0.1):
    """Exact solitary wave of u_t + a u u_x + b u_xxx - c u_xxxxx = 0 (data for the K* targets):
    u = 105 b^2/(169 a c) sech^4( sqrt(b/(13 c))/2 (x - x0 - 36 b^2 t/(169 c)) )."""
    a, b, c = w.adv, w.disp3, w.disp5
    A = 105.0 * b * b / (169.0 * a * c)
    kap = 0.5 * math.sqrt(b / (13.0 * c))
    V = 36.0 * b * b / (169.0 * c)
    return A / np.cosh(kap * (np.asarray(x, np.float64) - x0 - V * np.asarray(t, np.float64))) ** 4


def aniso_forcing(P, w: Workload):
    """f = sum_{a<=b} K_ab d_a d_b u* of the manufactured u* = prod_a sin(pi x_a) (data for the A* sets)."""
    P = np.asarray(P, np.float64)
    D = P.shape[1]
    s, c = np.sin(np.pi * P), np.cos(np.pi * P)
    pairs = [(a, b) for a in range(D) for b in range(a, D)]
    f = np.zeros(len(P))
    for q, (a, b) in enumerate(pairs):
        if a == b:
            d2 = -np.pi ** 2 * np.prod(s, 1)
        else:
            rest = np.prod(np.delete(s, [a, b], axis=1), 1) if D > 2 else 1.0
            d2 = np.pi ** 2 * c[:, a] * c[:, b] * rest
        f += w.aniso[q] * d2
    return f


def make_points(w: Workload, seed: int = POINT_SEED) -> PointSet:
    rng = np.random.Generator(np.random.PCG64(seed))
    if w.pde == "kawahara":
        x = rng.uniform(-1.0, 1.0, size=w.n_int)
        t = rng.uniform(0.0, 1.0, size=w.n_int)
        nb = w.n_bnd // 2
        tb = np.linspace(0.0, 1.0, nb)
        bnd = _f32(np.concatenate([np.stack([-np.ones(nb), tb], 1), np.stack([np.ones(nb), tb], 1)], 0))
        x0 = np.linspace(-1.0, 1.0, w.n_ic)
        ic = _f32(np.stack([x0, np.zeros_like(x0)], 1))
        return PointSet(_f32(np.stack([x, t], 1)), bnd, _f32(kawahara_wave(bnd[:, 0], bnd[:, 1], w)), ic,
                        _f32(kawahara_wave(ic[:, 0], ic[:, 1], w)))
    if w.pde == "aniso":
        interior = _f32(rng.uniform(-1.0, 1.0, size=(w.n_int, w.D)))
        if w.D == 2:
            bnd = _edges_2d(w.n_bnd // 4)
        else:
            q = np.arange(w.n_bnd)
            bnd = rng.uniform(-1.0, 1.0, size=(w.n_bnd, 3))
            bnd[q, (q % 6) // 2] = np.where(q % 2 == 0, -1.0, 1.0)
        return PointSet(interior, _f32(bnd), np.zeros(len(bnd), np.float32), forcing=_f32(aniso_forcing(interior, w)))
    if w.key.startswith("PP"):
        interior = rng.uniform(-1.0, 1.0, size=(w.n_int, 2))
        bnd = _edges_2d(w.n_bnd // 4)
        return PointSet(_f32(interior), _f32(bnd), np.zeros(len(bnd), np.float32))
    if w.key.startswith("PB"):
        interior = rng.uniform(w.lo, w.hi, size=(w.n_int, 2))
        nb = w.n_bnd // 2
        tb = np.linspace(w.lo, w.hi, nb)
        bnd = np.concatenate([np.stack([np.full(nb, w.lo), tb], 1), np.stack([np.full(nb, w.hi), tb], 1)], 0)
        y0 = np.linspace(w.lo, w.hi, w.n_ic)
        ic32 = _f32(np.stack([y0, np.zeros_like(y0)], 1))
        g0 = _f32(1.0 / np.cosh(4.0 * ic32[:, 0].astype(np.float64) - 5.0))   # u(y,0) = 1/cosh(4y-5)
        return PointSet(_f32(interior), _f32(bnd), np.zeros(len(bnd), np.float32), ic32, g0)
    if w.key.startswith("C1"):
        n = int(round(math.sqrt(w.n_int)))
        c = -1.0 + (2.0 * np.arange(n) + 1.0) / n            # cell-centred grid
        X, Y = np.meshgrid(c, c, indexing="ij")
        interior = np.stack([X.ravel(), Y.ravel()], 1)
        bnd = _edges_2d(w.n_bnd // 4)
        return PointSet(_f32(interior), _f32(bnd), np.zeros(len(bnd), np.float32))
    if w.pde == "poisson" and w.D == 2:
        interior = rng.uniform(-1.0, 1.0, size=(w.n_int, 2))
        bnd = _edges_2d(w.n_bnd // 4)
        return PointSet(_f32(interior), _f32(bnd), np.zeros(len(bnd), np.float32))
    if w.pde == "poisson" and w.D == 3:
        interior = rng.uniform(-1.0, 1.0, size=(w.n_int, 3))
        q = np.arange(w.n_bnd)
        face = q % 6
        bnd = rng.uniform(-1.0, 1.0, size=(w.n_bnd, 3))
        axis = face // 2
        side = np.where(face % 2 == 0, -1.0, 1.0)
        bnd[q, axis] = side
        return PointSet(_f32(interior), _f32(bnd), np.zeros(len(bnd), np.float32))
    if w.pde == "burgers":
        x = rng.uniform(-1.0, 1.0, size=w.n_int)
        t = rng.uniform(0.0, 1.0, size=w.n_int)
        interior = np.stack([x, t], 1)
        nb = w.n_bnd // 2
        tb = np.linspace(0.0, 1.0, nb)
        bnd = np.concatenate([np.stack([-np.ones(nb), tb], 1), np.stack([np.ones(nb), tb], 1)], 0)
        x0 = np.linspace(-1.0, 1.0, w.n_ic)
        ic = np.stack([x0, np.zeros_like(x0)], 1)
        ic32 = _f32(ic)
        g0 = _f32(-np.sin(np.pi * ic32[:, 0].astype(np.float64)))   # u(x,0) = -sin(pi x)
        return PointSet(_f32(interior), _f32(bnd), np.zeros(len(bnd), np.float32), ic32, g0)
    raise ValueError(w.key)


def random_params(widths, G: int, k: int, seed: int = PARAM_SEED, w_scale: float = 1.0,
                  bias_std: float = 0.0) -> List[tuple]:
    """W_l ~ N(0, w_scale^2 / (in*(G+k))) (variance reading, SURVEY.md §8(c) reading 5), b_l ~ N(0, bias_std^2).

    Returns a list of (W[O,I,B] float32, b[O] float32)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    B = G + k
    out = []
    for l in range(len(widths) - 1):
        I, O = widths[l], widths[l + 1]
        W = rng.standard_normal((O, I, B)) * (w_scale / math.sqrt(I * B))
        b = rng.standard_normal(O) * bias_std if bias_std > 0 else np.zeros(O)
        out.append((_f32(W), _f32(b)))
    return out


def flatten_params(params) -> np.ndarray:
    """Flat layout of include/hrkan.h: for each layer W[O][I][B] row-major, then b[O]."""
    return np.concatenate([np.concatenate([W.ravel(), b.ravel()]) for W, b in params]).astype(np.float32)


def unflatten_params(flat: np.ndarray, widths, B: int) -> List[tuple]:
    out, off = [], 0
    for l in range(len(widths) - 1):
        I, O = widths[l], widths[l + 1]
        W = flat[off:off + O * I * B].reshape(O, I, B)
        off += O * I * B
        b = flat[off:off + O]
        off += O
        out.append((W, b))
    assert off == len(flat)
    return out
