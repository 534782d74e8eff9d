import os, sys
sys.path.insert(0, os.getcwd())
import torch
import hrkan_inputs as HI
from paper_2409_14248_b200 import HRKANNet, pde_struct
for key in ["C1", "C2"]:
    w = HI.WORKLOADS[key]
    ps = HI.make_points(w)
    net = HRKANNet(w.widths, w.G, w.k, w.m, seed=HI.PARAM_SEED)
    cu = lambda a: None if a is None else torch.from_numpy(a).cuda()
    for _ in range(2):
        net.pinn_loss_grad(pde_struct(w.pde, w.alpha, w.adv, w.visc), cu(ps.interior), cu(ps.boundary), cu(ps.g_boundary), cu(ps.initial), cu(ps.g_initial))
    torch.cuda.synchronize()
print("ok")
