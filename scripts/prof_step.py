"""One PINN loss+grad step on a synthetic sample of a workload (for ncu captures of single kernels).

    python scripts/prof_step.py [C5] [n_interior=65536] [reps=2]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import hrkan_inputs as HI  # noqa: E402
from paper_2409_14248_b200 import HRKANNet, pde_struct  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "C5"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 16
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
w = HI.WORKLOADS[key]
net = HRKANNet(w.widths, w.G, w.k, w.m, seed=HI.PARAM_SEED)
pts = torch.rand(n, w.D, device="cuda") * 2 - 1
if w.pde == "burgers":
    pts[:, 1] = (pts[:, 1] + 1) / 2
nb = max(8, n // 256)
bnd = torch.rand(nb, w.D, device="cuda") * 2 - 1
gb = torch.zeros(nb, device="cuda")
pde = pde_struct(w.pde, w.alpha, w.adv, w.visc)
for _ in range(reps):
    out = net.pinn_loss_grad(pde, pts, bnd, gb)
torch.cuda.synchronize()
print("ok", key, n, float(out[-4:-2].sum()))
