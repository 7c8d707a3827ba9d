"""A/B timing of one library build (IGALR_PKG_ROOT env selects it): median CUDA-event time of the
mass+stiffness apply (and of the stiffness part alone) for the given configs."""
import os
import statistics
import sys

# IGALR_PKG_ROOT: an experiment package root laid out by tools/mkvariant.sh (default: the repo)
sys.path.insert(0, os.path.abspath(os.environ.get("IGALR_PKG_ROOT") or
                                   os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1811_06797_b200 import workloads  # noqa: E402


def t_apply(fn, s, reps=30):
    for _ in range(3):
        fn()
    s.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        fn()
        e1.record(s)
        s.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


tag = os.environ.get("IGALR_PKG_ROOT", "default") or "default"
for name in (sys.argv[1:] or ["c3", "c5"]):
    cfg = synth.CONFIGS[name]
    op = workloads.build_operator(cfg, synth.draw_weights(cfg))
    nx, ny, nz = op.info_dict()["dims"]
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        if cfg.kkt:
            x = torch.randn((3, cfg.n_t, nz, ny, nx), dtype=torch.float64, device="cuda")
            y = torch.empty_like(x)
            full = t_apply(lambda: op.kkt_apply(x, y, cfg.n_t, cfg.tau, cfg.beta, stream=s), s)
            print("%-8s %s kkt %.4f ms" % (name, os.path.basename(tag), full))
            continue
        g = torch.Generator(device="cuda")
        g.manual_seed(1234)
        x = torch.randn((cfg.batch, nz, ny, nx), dtype=torch.float64, device="cuda", generator=g)
        y1, y2 = torch.empty_like(x), torch.empty_like(x)
        full = t_apply(lambda: op.apply(x, y1, y2, stream=s), s)
        stiff = t_apply(lambda: op.apply(x, None, y2, stream=s), s)
        mass = t_apply(lambda: op.apply(x, y1, None, stream=s), s)
    # (A/B sanity: output fingerprints of the same seeded input; builds that differ only in summation
    # order agree to ~1e-15 relative)
    w = torch.linspace(1.0, 2.0, x.numel(), dtype=torch.float64, device="cuda").view_as(x)
    print("%-8s %s full %.4f ms  stiff %.4f  mass %.4f  | fp mass %.15e stiff %.15e" %
          (name, os.path.basename(tag), full, stiff, mass, float((y1 * w).sum()), float((y2 * w).sum())))
