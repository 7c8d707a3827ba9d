"""Run one workload's apply a few times (for ncu / compute-sanitizer captures)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1811_06797_b200 import workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--path", default="auto")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--batch", type=int, default=None)
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]
if a.n or a.batch:
    cfg = synth.scaled(cfg, a.n or cfg.n, batch=a.batch or cfg.batch)
w = synth.draw_weights(cfg)
op = workloads.build_operator(cfg, w)
nx, ny, nz = cfg.dims
shape = (3, cfg.n_t, nz, ny, nx) if cfg.kkt else (cfg.batch, nz, ny, nx)
x = torch.randn(shape, dtype=torch.float64, device="cuda")
y1, y2 = torch.empty_like(x), torch.empty_like(x)
for _ in range(a.reps):
    if cfg.kkt:
        op.kkt_apply(x, y1, cfg.n_t, cfg.tau, cfg.beta, path=a.path)
    else:
        op.apply(x, y1, y2, path=a.path)
torch.cuda.synchronize()
print("ok", op.info_dict())
