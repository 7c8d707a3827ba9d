import sys, os
sys.path.insert(0, os.getcwd())
import torch, synth
from paper_1811_06797_b200 import workloads
cfg = synth.CONFIGS["c4"]; op = workloads.build_operator(cfg, synth.draw_weights(cfg))
mx, my, mz = op.dims; R1 = R2 = 20
gz = torch.randn((mz, R1), dtype=torch.float64, device="cuda"); gy = torch.randn((R1, my, R2), dtype=torch.float64, device="cuda"); gx = torch.randn((R2, mx), dtype=torch.float64, device="cuda")
T = len(op.terms(1)[1]); L = torch.empty((T, R1, R1), dtype=torch.float64, device="cuda"); R = torch.empty((T, R2, R2), dtype=torch.float64, device="cuda")
x = torch.randn((R1, my, R2), dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
op.tt_interfaces(1, 1, gz, gy, gx, L, R)
for _ in range(3): op.tt_local_apply(1, 1, L, R, x, y)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(20): op.tt_local_apply(1, 1, L, R, x, y)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=10, max_name_column_width=50))
