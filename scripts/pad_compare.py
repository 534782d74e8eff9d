"""Width padding A/B (hrkan_create pads hidden widths in (32, 256] to 64/128/256 so every hidden->hidden
layer runs on the tensor cores): loss+grad device time of nets with off-size hidden widths, padded
(default) vs HRKAN_PAD_WIDTHS=0 (the band-limited SIMT kernels on the caller's widths).
    python scripts/pad_compare.py [--n 65536] [--reps 3]"""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2409_14248_b200 import HRKANNet, pde_struct  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1 << 16)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
NETS = [((2, 100, 100, 1), 10, "poisson"), ((2, 48, 48, 1), 10, "poisson"), ((2, 96, 96, 96, 1), 8, "burgers"),
        ((3, 200, 200, 1), 16, "poisson"), ((2, 64, 64, 1), 10, "poisson")]
for widths, G, kind in NETS:
    row = []
    for pad in ("1", "0"):
        os.environ["HRKAN_PAD_WIDTHS"] = pad
        net = HRKANNet(widths, G, 3, 4, seed=3)
        D = widths[0]
        g = torch.Generator(device="cpu").manual_seed(1)
        pts = (torch.rand(a.n, D, generator=g) * 2 - 1).cuda()
        if kind == "burgers":
            pts[:, 1] = (pts[:, 1] + 1) / 2
        pde = pde_struct(kind, 0.05, 1.0, 0.01)
        bnd = pts[: a.n // 16].clone()
        gb = torch.zeros(a.n // 16, device="cuda")
        out = net.pinn_loss_grad(pde, pts, bnd, gb)
        torch.cuda.synchronize()
        ts = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            out = net.pinn_loss_grad(pde, pts, bnd, gb)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        row.append((statistics.median(ts), float(out[-4]), float(out[-3])))
        del net
    (tp, lp, bp), (tu, lu, bu) = row
    print(f"{'x'.join(map(str, widths)):>16s} G={G} {kind:8s} n={a.n}: padded {tp:8.3f} ms  unpadded {tu:8.3f} ms  "
          f"speed-up {tu / tp:5.2f}x   loss parts padded ({lp:.6g}, {bp:.6g}) unpadded ({lu:.6g}, {bu:.6g})", flush=True)
