"""Per-layer / per-engine error breakdown of test_gpu_regressions' randomized stress cases (debug aid)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import hrkan_inputs as HI  # noqa: E402
from test_gpu_regressions import _stress_cases  # noqa: E402
from test_gpu_parity import _loss_grad_gpu, _loss_grad_oracle, _make, rel_l2  # noqa: E402
from oracle import hrkan_oracle as O  # noqa: E402

sel = [int(a) for a in sys.argv[1:]] or None
for case in _stress_cases():
    q, D, O_, depth, G, k, m, pde, n_int, n_bi, chunk = case
    if sel and q not in sel:
        continue
    widths = (D,) + (O_,) * depth + (1,)
    w = HI.Workload(f"S{q}", "stress", pde, widths, G, k, m, n_int, n_bi, 0, adv=0.7 if pde == "burgers" else 1.0, visc=0.02)
    rng = np.random.default_rng(q)
    interior = rng.uniform(-1, 1, (n_int, D))
    if pde == "burgers":
        interior[:, 1] = rng.uniform(0, 1, n_int)
    bnd = rng.uniform(-1, 1, (n_bi, D))
    if n_bi:
        bnd[:, 0] = np.where(rng.random(n_bi) < 0.5, -1.0, 1.0)
    ps = HI.PointSet(interior.astype(np.float32), bnd.astype(np.float32), rng.uniform(-0.5, 0.5, n_bi).astype(np.float32))
    lp, lb, g = _loss_grad_oracle(w, HI.random_params(w.widths, w.G, w.k, seed=100 + q, bias_std=0.1), ps)
    print(f"case {case}: oracle lp {lp:.6g} lb {lb:.6g}")
    for engine in (0, 1):
        try:
            net, params = _make(w, seed=100 + q, chunk=chunk, engine=engine)
            out = _loss_grad_gpu(torch, net, w, ps)
        except Exception as e:
            print(f"  engine {engine}: ERROR {e}")
            continue
        npar = w.num_params()
        gl = HI.unflatten_params(out[:npar].copy(), w.widths, w.B)
        errs = [(round(rel_l2(a, c), 6), round(rel_l2(b, d), 6)) for (a, b), (c, d) in zip(gl, g)]
        print(f"  engine {engine}: lp {out[npar]:.6g} lb {out[npar+1]:.6g} flag {out[npar+2]} total {rel_l2(out[:npar], O.flat_grad(g)):.3g} per-layer (dW, db) {errs}")
    u, du, d2u = [t.cpu().numpy() for t in _make(w, seed=100 + q, chunk=chunk)[0].forward_jet(torch.from_numpy(ps.interior).cuda())]
    ou, odu, od2u = O.forward_jet(O.Net(w.widths, w.G, w.k, w.m), params, ps.interior)
    print(f"  forward: u {rel_l2(u, ou):.3g} du {rel_l2(du, odu):.3g} d2u {rel_l2(d2u, od2u):.3g}")
