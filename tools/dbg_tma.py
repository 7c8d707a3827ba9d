import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_1811_06797_b200 import workloads
cfgname, n, part = sys.argv[1], int(sys.argv[2]), sys.argv[3]
cfg = synth.scaled(synth.CONFIGS[cfgname], n, batch=1)
w = synth.draw_weights(cfg)
op = workloads.build_operator(cfg, w, mass=(part != "s"), stiff=(part != "m"))
x = torch.randn((1, n, n, n), dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
if part == "m": op.apply(x, y, None, path="fused")
else: op.apply(x, None, y, path="fused")
torch.cuda.synchronize()
print("OK", cfgname, n, part, os.environ.get("IGALR_QX"), os.environ.get("IGALR_YRES"))
