"""Per-kernel-class device time of one loss+grad call (median of reps), for same-box A/B runs of
library variants (HRKAN_LIB=...):  python scripts/ab_time.py [C5 C4 C3] [--n 262144] [--reps 5]"""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import hrkan_inputs as HI  # noqa: E402
from paper_2409_14248_b200 import HRKANNet, pde_struct  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("keys", nargs="*", default=["C5", "C4", "C3"])
ap.add_argument("--n", type=int, default=1 << 18)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--m", type=int, default=0, help="override the HR order m (0: the workload's)")
ap.add_argument("--engine", type=int, default=0, help="0 auto, 1 band-limited SIMT, 2 tensor cores")
a = ap.parse_args()
tag = os.path.basename(os.path.dirname(os.environ.get("HRKAN_LIB", "/base/x")))
for key in a.keys:
    w = HI.WORKLOADS[key]
    net = HRKANNet(w.widths, w.G, w.k, a.m or w.m, seed=HI.PARAM_SEED)
    net.set_engine(a.engine)
    g = torch.Generator(device="cpu").manual_seed(1)
    pts = (torch.rand(a.n, w.D, generator=g) * 2 - 1).cuda()
    if w.pde == "burgers":
        pts[:, 1] = (pts[:, 1] + 1) / 2
    pde = pde_struct(w.pde, w.alpha, w.adv, w.visc)
    nb = a.n // 16
    bnd = pts[:nb].clone()
    gb = torch.zeros(nb, device="cuda")
    net.pinn_loss_grad(pde, pts, bnd, gb)
    torch.cuda.synchronize()
    tot, cls = [], {}
    for r in range(a.reps):
        net.profile_enable(True)
        net.profile_read()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        net.pinn_loss_grad(pde, pts, bnd, gb)
        e1.record()
        torch.cuda.synchronize()
        pr = net.profile_read()
        net.profile_enable(False)
        tot.append(e0.elapsed_time(e1))
        for k, v in pr.items():
            cls.setdefault(k, []).append(v[0])
    med = {k: round(statistics.median(v), 3) for k, v in cls.items() if statistics.median(v) > 0.05}
    print(f"{tag:10s} {key} m={a.m or w.m} eng={a.engine} total {statistics.median(tot):.3f} ms", med, flush=True)
