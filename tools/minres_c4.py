"""c4 all-at-once KKT solve: preconditioned MINRES iterations / time (NEXT-1 measurement)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_1811_06797_b200 import workloads
cfg = synth.CONFIGS["c4"]
w = synth.draw_weights(cfg)
op = workloads.build_operator(cfg, w)
m = cfg.n - 2
g = torch.Generator(device="cuda").manual_seed(7)
yhat = torch.randn((cfg.n_t, m, m, m), dtype=torch.float64, device="cuda", generator=g)
b = torch.zeros((3, cfg.n_t, m, m, m), dtype=torch.float64, device="cuda")
ym = torch.empty_like(yhat)
op.apply(yhat, ym, None)
b[0] = cfg.tau * ym
t0 = time.time(); prec = op.kkt_preconditioner(cfg.n_t, cfg.tau, cfg.beta); torch.cuda.synchronize(); t1 = time.time()
print("prec setup s", round(t1 - t0, 3), "mbar/sbar", prec.info()[:2])
for rtol in (1e-6, 1e-8, 1e-10):
    x = torch.empty_like(b)
    torch.cuda.synchronize(); t0 = time.time()
    info = op.kkt_minres(b, x, cfg.n_t, cfg.tau, cfg.beta, rtol=rtol, maxit=3000, prec=prec)
    torch.cuda.synchronize(); t1 = time.time()
    ax = torch.empty_like(b); op.kkt_apply(x, ax, cfg.n_t, cfg.tau, cfg.beta)
    r2 = float(torch.linalg.vector_norm(b - ax) / torch.linalg.vector_norm(b))
    print("rtol", rtol, "iters", info.iters, "conv", info.converged, "s", round(t1 - t0, 3), "ms/iter", round(1e3 * (t1 - t0) / max(info.iters, 1), 3), "rel2", r2)
x = torch.empty_like(b)
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
s = torch.cuda.current_stream()
e0.record(s); info = op.kkt_minres(b, x, cfg.n_t, cfg.tau, cfg.beta, rtol=0.0, maxit=20, prec=prec); e1.record(s); torch.cuda.synchronize()
print("20 iters ms/iter (events)", e0.elapsed_time(e1) / 20)
r = torch.randn_like(b); o = torch.empty_like(b)
for _ in range(3): prec.apply(r, o)
e0.record(s)
for _ in range(20): prec.apply(r, o)
e1.record(s); torch.cuda.synchronize(); print("prec apply ms", e0.elapsed_time(e1) / 20)
for _ in range(3): op.kkt_apply(r, o, cfg.n_t, cfg.tau, cfg.beta)
e0.record(s)
for _ in range(20): op.kkt_apply(r, o, cfg.n_t, cfg.tau, cfg.beta)
e1.record(s); torch.cuda.synchronize(); print("kkt apply ms", e0.elapsed_time(e1) / 20)
