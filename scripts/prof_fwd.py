import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import hrkan_inputs as HI
from paper_2409_14248_b200 import HRKANNet
key = sys.argv[1] if len(sys.argv) > 1 else "C5"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 16
w = HI.WORKLOADS[key]
net = HRKANNet(w.widths, w.G, w.k, w.m)
net.set_engine(2)
pts = torch.rand(n, w.D, device="cuda") * 2 - 1
for _ in range(2):
    net.forward_jet(pts)
torch.cuda.synchronize()
print("ok")
