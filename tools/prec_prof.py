"""Per-kernel breakdown of the c4 KKT preconditioner apply and PMINRES iterations (torch.profiler)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import synth  # noqa: E402
from paper_1811_06797_b200 import workloads  # noqa: E402
cfg = synth.CONFIGS["c4"]
op = workloads.build_operator(cfg, synth.draw_weights(cfg))
m = cfg.n - 2
b = torch.randn((3, cfg.n_t, m, m, m), dtype=torch.float64, device="cuda")
x = torch.empty_like(b)
prec = op.kkt_preconditioner(cfg.n_t, cfg.tau, cfg.beta)
op.kkt_minres(b, x, cfg.n_t, cfg.tau, cfg.beta, rtol=0.0, maxit=3, prec=prec)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as p:
    op.kkt_minres(b, x, cfg.n_t, cfg.tau, cfg.beta, rtol=0.0, maxit=20, prec=prec)
    torch.cuda.synchronize()
print(p.key_averages().table(sort_by="cuda_time_total", row_limit=14, max_name_column_width=60))
