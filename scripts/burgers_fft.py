"""Ground truth of the paper's viscous Burgers experiment by a Fourier pseudo-spectral solve
(Sec. 4.2: "We solve for the ground-truth solution using Fast Fourier Transform
method"), used only to score the trained networks of scripts/train_paper_burgers.py.

Original problem:  u_t + u u_x - nu u_xx = 0 on x in [-5, 5], t in [0, 2.5],
u(+-5, t) = 0, u(x, 0) = 1/cosh(x), nu = 0.001.  The paper trains on the transformed variable
y = (x + 5)/4 in [0, 2.5]; the test grid is 200 x 200 over (y, t).

Method: the domain is treated as periodic (1/cosh(5) = 0.013, so the boundary mismatch is small and
confined to the edges), N Fourier modes, integrating-factor RK4 in time (the viscous term exactly,
the conservative flux -(u^2/2)_x pseudo-spectrally with 2/3 de-aliasing).  Plain numpy float64.

    python scripts/burgers_fft.py [--n 8192] [--dt 5e-5]      # self-check (refinement + mass)
"""
import argparse

import numpy as np

NU = 0.001
X_LO, X_HI = -5.0, 5.0
T_END = 2.5


def solve(times, n=8192, dt=5e-5, nu=NU):
    """u(x_j, t) on the periodic grid x_j = X_LO + j*L/n for each t in `times` (sorted, <= T_END)."""
    L = X_HI - X_LO
    x = X_LO + L * np.arange(n) / n
    k = 2.0 * np.pi * np.fft.rfftfreq(n, d=L / n)
    dealias = np.abs(k) < (2.0 / 3.0) * k.max()
    u_hat = np.fft.rfft(1.0 / np.cosh(x))
    lin = -nu * k * k
    e_half, e_full = np.exp(lin * dt / 2), np.exp(lin * dt)

    def flux(vh):                                   # FFT of -(u^2 / 2)_x, de-aliased
        u = np.fft.irfft(vh * dealias, n)
        return -0.5j * k * np.fft.rfft(u * u) * dealias

    out, t, ti = [], 0.0, 0
    times = list(times)
    while ti < len(times):
        while ti < len(times) and times[ti] <= t + 1e-12:
            out.append(np.fft.irfft(u_hat, n))
            ti += 1
        if ti >= len(times):
            break
        h = min(dt, times[ti] - t)
        eh, ef = (e_half, e_full) if h == dt else (np.exp(lin * h / 2), np.exp(lin * h))
        a = flux(u_hat)
        b = flux(eh * (u_hat + 0.5 * h * a))
        c = flux(eh * u_hat + 0.5 * h * b)
        d = flux(ef * u_hat + h * eh * c)
        u_hat = ef * u_hat + (h / 6.0) * (ef * a + 2.0 * eh * (b + c) + d)
        t += h
    return x, np.array(out)


def test_grid(ny=200, nt=200, n=8192, dt=5e-5):
    """The paper's 200 x 200 test grid over the transformed (y, t) in [0, 2.5]^2 and the ground truth
    there (the periodic solution interpolated linearly in x = 4y - 5)."""
    y = np.linspace(0.0, 2.5, ny)
    t = np.linspace(0.0, T_END, nt)
    x, U = solve(t, n=n, dt=dt)
    xq = 4.0 * y - 5.0
    xp = np.concatenate([x, [X_HI]])
    truth = np.stack([np.interp(xq, xp, np.concatenate([U[j], U[j][:1]])) for j in range(nt)], 1)   # [ny][nt]
    Y, T = np.meshgrid(y, t, indexing="ij")
    return np.stack([Y.ravel(), T.ravel()], 1), truth.ravel()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--dt", type=float, default=5e-5)
    a = ap.parse_args()
    times = [0.0, 1.0, 2.0, 2.5]
    x, U = solve(times, a.n, a.dt)
    _, U2 = solve(times, a.n, a.dt / 2)
    xh, Uh = solve(times, 2 * a.n, a.dt / 2)
    dx = (X_HI - X_LO) / a.n
    for j, t in enumerate(times):
        print(f"t={t:4.2f}  mass {U[j].sum() * dx:.10f}  max|u| {np.abs(U[j]).max():.6f}  "
              f"dt/2 diff {np.abs(U[j] - U2[j]).max():.2e}  2n diff {np.abs(U[j] - Uh[j][::2]).max():.2e}")


if __name__ == "__main__":
    main()
