"""Aggregate the per-warp cycle accounting of an IGALR_EXP_TIMERS build (tools/mkvariant.sh <tag>
"-DIGALR_EXP_FAST -DIGALR_EXP_TIMERS"): one mass-only and one stiffness-only apply, the kernel's
EXPT lines (device printf) averaged over the sampled warps, as shares of the warp's total.
usage: IGALR_PKG_ROOT=exp/<tag> python tools/exp_timers.py [config]"""
import os
import re
import subprocess
import sys

if os.environ.get("EXPT_CHILD"):
    sys.path.insert(0, os.path.abspath(os.environ.get("IGALR_PKG_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
    import torch
    import synth
    from paper_1811_06797_b200 import workloads
    cfg = synth.CONFIGS[sys.argv[1]]
    op = workloads.build_operator(cfg, synth.draw_weights(cfg))
    nx, ny, nz = op.info_dict()["dims"]
    x = torch.randn((cfg.batch, nz, ny, nx), dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    if sys.argv[2] == "mass":
        op.apply(x, y, None)
    else:
        op.apply(x, None, y)
    torch.cuda.synchronize()
    sys.exit(0)

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
for part in ("mass", "stiff"):
    out = subprocess.run([sys.executable, __file__, name, part], env=dict(os.environ, EXPT_CHILD="1"),
                         capture_output=True, text=True).stdout
    rows = []
    for line in out.splitlines():
        if line.startswith("EXPT"):
            kv = re.findall(r"(\w+) (-?\d+)", line)
            rows.append({k: int(v) for k, v in kv})
    if not rows:
        print(part, "no EXPT lines")
        continue
    keys = [k for k in rows[0] if k not in ("cta", "warp")]
    tot = sum(r["total"] for r in rows) / len(rows)
    print("%s %s: %d warps, mean total %.0f cycles" % (name, part, len(rows), tot))
    print("  " + "  ".join("%s %.1f%%" % (k, 100.0 * sum(r[k] for r in rows) / len(rows) / tot) for k in keys if k != "total"))
