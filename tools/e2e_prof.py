import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch, synth
from paper_1811_06797_b200 import workloads
cfg = synth.CONFIGS["c3"]; knots, w, x = synth.draw_problem(cfg)
op = workloads.build_operator(cfg, w)
xh = torch.from_numpy(x).pin_memory(); ymh = torch.empty_like(xh).pin_memory(); ysh = torch.empty_like(xh).pin_memory()
xn, ymn, ysn = xh.numpy(), ymh.numpy(), ysh.numpy()
for b in (1, 2, 8):
    op.apply_host(xn[:b], ymn[:b], ysn[:b])
    t0 = time.perf_counter()
    for _ in range(5): op.apply_host(xn[:b], ymn[:b], ysn[:b])
    dt = (time.perf_counter() - t0) / 5
    print("batch", b, "ms", round(dt * 1e3, 3), "GDoF/s", round(b * x[0].size / dt / 1e9, 3))
# raw PCIe rates with pinned memory
d = torch.empty_like(xh[:4], device="cuda")
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(5): d.copy_(xh[:4], non_blocking=True)
torch.cuda.synchronize(); print("H2D GB/s", 5 * xh[:4].numel() * 8 / (time.perf_counter() - t0) / 1e9)
t0 = time.perf_counter()
for _ in range(5): ymh[:4].copy_(d, non_blocking=True)
torch.cuda.synchronize(); print("D2H GB/s", 5 * xh[:4].numel() * 8 / (time.perf_counter() - t0) / 1e9)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
d2 = torch.empty_like(d)
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(5):
    with torch.cuda.stream(s1): d.copy_(xh[:4], non_blocking=True)
    with torch.cuda.stream(s2): ymh[:4].copy_(d2, non_blocking=True)
torch.cuda.synchronize(); print("duplex GB/s each", 5 * xh[:4].numel() * 8 / (time.perf_counter() - t0) / 1e9)
