"""Per-kernel device time breakdown of repeated applies / KKT matvecs (torch.profiler / CUPTI)."""
import argparse
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import synth  # noqa: E402
from paper_1811_06797_b200 import workloads  # noqa: E402
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--path", default="auto")
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]
op = workloads.build_operator(cfg, synth.draw_weights(cfg))
nx, ny, nz = op.info_dict()["dims"]
s = torch.cuda.Stream()
if cfg.kkt:
    x = torch.randn((3, cfg.n_t, nz, ny, nx), dtype=torch.float64, device="cuda")
    y1 = torch.empty_like(x)
    step = lambda: op.kkt_apply(x, y1, cfg.n_t, cfg.tau, cfg.beta, stream=s, path=a.path)
else:
    x = torch.randn((cfg.batch, nz, ny, nx), dtype=torch.float64, device="cuda")
    y1, y2 = torch.empty_like(x), torch.empty_like(x)
    step = lambda: op.apply(x, y1, y2, stream=s, path=a.path)
for _ in range(3):
    step()
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(a.reps):
        step()
    e1.record(s)
    torch.cuda.synchronize()
print(a.config, "event ms/step", e0.elapsed_time(e1) / a.reps)
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=12, max_name_column_width=70))
