"""Per-kernel device time breakdown of repeated applies (torch.profiler / CUPTI)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_1811_06797_b200 import workloads
ap = argparse.ArgumentParser(); ap.add_argument("--config", default="c3"); ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--path", default="auto")
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]; w = synth.draw_weights(cfg); op = workloads.build_operator(cfg, w)
nx, ny, nz = cfg.dims
x = torch.randn((cfg.batch, nz, ny, nx), dtype=torch.float64, device="cuda"); y1, y2 = torch.empty_like(x), torch.empty_like(x)
s = torch.cuda.Stream()
for _ in range(3): op.apply(x, y1, y2, stream=s, path=a.path)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(a.reps): op.apply(x, y1, y2, stream=s, path=a.path)
    e1.record(s); torch.cuda.synchronize()
print("event ms/step", e0.elapsed_time(e1) / a.reps)
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=12, max_name_column_width=60))
