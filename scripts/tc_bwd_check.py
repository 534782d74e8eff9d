"""GPU check: tcgen05 dgrad/wgrad (engine 2) vs SIMT (engine 1) vs oracle, and per-class timing."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import hrkan_inputs as HI
from oracle import hrkan_oracle as O
from paper_2409_14248_b200 import HRKANNet, pde_struct

def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-300))

keys = sys.argv[1:] or ["C5", "C4"]
for key in keys:
    w = HI.WORKLOADS[key]
    ps = HI.make_points(w).subset(8192 if key == "C5" else 1024, 256 if key == "C5" else 64)
    params = HI.random_params(w.widths, w.G, w.k, seed=7, bias_std=0.1)
    cu = lambda a: None if a is None else torch.from_numpy(a).cuda()
    outs = {}
    for eng in (1, 2):
        net = HRKANNet(w.widths, w.G, w.k, w.m)
        net.set_params(HI.flatten_params(params))
        net.set_engine(eng)
        out = net.pinn_loss_grad(pde_struct(w.pde, w.alpha, w.adv, w.visc), cu(ps.interior), cu(ps.boundary),
                                 cu(ps.g_boundary), cu(ps.initial), cu(ps.g_initial))
        torch.cuda.synchronize()
        outs[eng] = out.cpu().numpy()
    bi = ps.boundary if ps.initial is None else np.concatenate([ps.boundary, ps.initial])
    gbi = ps.g_boundary if ps.initial is None else np.concatenate([ps.g_boundary, ps.g_initial])
    lp, lb, g = O.loss_grad(O.Net(w.widths, w.G, w.k, w.m), params,
                            {"kind": w.pde, "alpha": w.alpha, "adv": w.adv, "visc": w.visc}, ps.interior, bi, gbi)
    flat = O.flat_grad(g)
    npar = w.num_params()
    ou, odu, od2u = O.forward_jet(O.Net(w.widths, w.G, w.k, w.m), params, ps.interior[:2048])
    for eng in (1, 2):
        net = HRKANNet(w.widths, w.G, w.k, w.m)
        net.set_params(HI.flatten_params(params))
        net.set_engine(eng)
        gu, gdu, gd2u = [t.cpu().numpy() for t in net.forward_jet(torch.from_numpy(ps.interior[:2048]).cuda())]
        print(key, "engine", eng, "forward u %.2e du %.2e d2u %.2e" % (rel(gu, ou), rel(gdu, odu), rel(gd2u, od2u)), flush=True)
    for eng in (1, 2):
        o = outs[eng]
        gl = HI.unflatten_params(o[:npar].copy(), w.widths, w.B)
        per = [(rel(a[0], b[0]), rel(a[1], b[1])) for a, b in zip(gl, g)]
        print(key, "engine", eng, "loss", rel([o[npar]], [lp]), rel([o[npar + 1]], [lb]), "grad", rel(o[:npar], flat),
              "per-layer", ["%.1e/%.1e" % x for x in per], "flag", o[npar + 2], flush=True)

for key in keys:
    w = HI.WORKLOADS[key]
    n = 1 << 18
    pts = (torch.rand(n, w.D, device="cuda") * 2 - 1).contiguous()
    if w.pde == "burgers":
        pts[:, 1] = (pts[:, 1] + 1) / 2
    bnd = torch.rand(n // 64, w.D, device="cuda") * 2 - 1
    gb = torch.zeros(n // 64, device="cuda")
    for eng in (1, 2):
        net = HRKANNet(w.widths, w.G, w.k, w.m)
        net.set_engine(eng)
        pde = pde_struct(w.pde, w.alpha, w.adv, w.visc)
        net.pinn_loss_grad(pde, pts, bnd, gb); torch.cuda.synchronize()
        net.profile_enable(True); net.profile_read()
        t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
        t0.record(); net.pinn_loss_grad(pde, pts, bnd, gb); t1.record(); torch.cuda.synchronize()
        prof = {k: round(v[0], 3) for k, v in net.profile_read().items() if v[1]}
        print(key, "engine", eng, "loss_grad ms", round(t0.elapsed_time(t1), 3), prof, flush=True)
