"""Quick GPU check: tcgen05 forward hidden layer vs SIMT engine vs oracle (forward_jet)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import hrkan_inputs as HI
from oracle import hrkan_oracle as O
from paper_2409_14248_b200 import HRKANNet

def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-300))

for key in sys.argv[1:] or ["C5", "C4"]:
    w = HI.WORKLOADS[key]
    ps = HI.make_points(w).subset(4096 if key == "C5" else 1024, 64)
    pts = ps.interior[:777]
    params = HI.random_params(w.widths, w.G, w.k, seed=7, bias_std=0.1)
    res = {}
    for eng in (1, 2):
        net = HRKANNet(w.widths, w.G, w.k, w.m)
        net.set_params(HI.flatten_params(params))
        net.set_engine(eng)
        out = net.forward_jet(torch.from_numpy(pts).cuda())
        torch.cuda.synchronize()
        res[eng] = [t.cpu().numpy() for t in out]
    ou, odu, od2u = O.forward_jet(O.Net(w.widths, w.G, w.k, w.m), params, pts)
    for eng in (1, 2):
        u, du, d2u = res[eng]
        print(key, "engine", eng, "u", rel(u, ou), "du", rel(du, odu), "d2u", rel(d2u, od2u), flush=True)
    print(key, "tc vs simt u", rel(res[2][0], res[1][0]), "first u", res[2][0][:4], res[1][0][:4], flush=True)

# timing of forward_jet at scale (engine 1 = SIMT, 2 = tcgen05)
for key in sys.argv[1:] or ["C5", "C4"]:
    w = HI.WORKLOADS[key]
    n = 1 << 18
    pts = torch.rand(n, w.D, device="cuda") * 2 - 1
    for eng in (1, 2):
        net = HRKANNet(w.widths, w.G, w.k, w.m)
        net.set_engine(eng)
        net.forward_jet(pts); torch.cuda.synchronize()
        net.profile_enable(True); net.profile_read()
        t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
        t0.record(); net.forward_jet(pts); t1.record(); torch.cuda.synchronize()
        prof = {k: v for k, v in net.profile_read().items() if v[1]}
        C = 1 + 2 * w.D
        fl = 0
        for l in range(1, len(w.widths) - 2):
            fl += 2 * C * w.widths[l] * w.widths[l + 1] * w.B * n
        hid = prof.get("fwd_hidden", (0, 0))[0]
        print(key, "engine", eng, "forward_jet ms", t0.elapsed_time(t1), "hidden ms", hid,
              "hidden TFLOP/s (dense algorithmic)", fl / (hid / 1e3) / 1e12 if hid else None, flush=True)
