#!/usr/bin/env python
"""bench.py — GDoF/s of the fp64 low-rank Kronecker operator apply on B200 (+ % of roofline).

Default workload: BASELINE config c3 (128^3, p=3, R=8, mass + full anisotropic stiffness,
batch of 8 N(0,1) vectors) — the first full-size config the >= 70 % roofline target is
quoted on.  A "step" = one mass+stiffness apply (steps A6-A8 of SURVEY §8(a)) of the whole
batch; factor assembly (A1-A5) runs once before timing and is reported as setup_ms.  The other
configs (c2, c4 KKT, c5) are timed the same way and reported under "configs".

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]

Multi-GPU (torchrun, one process per GPU): every rank applies its own batch (weak scaling, the
batch dimension shards with no collective); time = max over ranks.
--impl reference times the CPU oracle (CSR SpMV of a one-plane row sample of the same workload,
the assembled full-size matrices' rows) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

PEAK_FP64_TFLOPS = 37.0  # measured: tools/ubench.cu DMMA/DFMA (profiles/r01_ubench.md); nominal 37.2 @1965 MHz


def _measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region by a background thread that
    polls NVML every `period_s` (2 ms: a 20-step c3 region of ~30 ms still gets ~15 samples).
    Falls back to `nvidia-smi -lms 10` when NVML is unavailable."""

    _REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
                "sw_power_cap": 0x4}

    def __init__(self, index: int, period_s: float = 0.002):
        self.index = index
        self.period = period_s
        self.rows = []  # (sm_mhz, sm_max_mhz, power_w, reasons bitmask)
        self.proc = None
        self.stop = threading.Event()
        self.t = None
        self.source = "nvml"

    def _poll_nvml(self, nv, h):
        while not self.stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
                pw = nv.nvmlDeviceGetPowerUsage(h) / 1000.0
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h) if hasattr(
                    nv, "nvmlDeviceGetCurrentClocksEventReasons") else nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                self.rows.append((float(sm), float(mx), pw, int(rs)))
            except Exception:
                pass
            self.stop.wait(self.period)

    def _read_smi(self):
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in self.proc.stdout:
            r = [v.strip() for v in line.split(",")]
            try:
                bits = sum(self._REASONS[n] for i, n in enumerate(names) if r[3 + i] == "Active")
                self.rows.append((float(r[0]), float(r[1]), float(r[2]), bits))
            except Exception:
                pass

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.t = threading.Thread(target=self._poll_nvml, args=(nv, h), daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.rows and time.time() - t0 < 2.0:
                time.sleep(0.001)
            self.rows = []
            return self
        except Exception:
            pass
        self.source = "nvidia-smi"
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "10"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read_smi, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.rows and time.time() - t0 < 5.0:
                time.sleep(0.01)
            self.rows = []
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.stop.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.t:
            self.t.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "source": self.source}
        sm = [r[0] for r in self.rows]
        reasons = sorted({n for r in self.rows for n, b in self._REASONS.items() if r[3] & b})
        return {"sm_mhz": statistics.median(sm), "sm_min_mhz": min(sm), "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": reasons, "power_w_max": max(r[2] for r in self.rows), "samples": len(self.rows),
                "source": self.source}


def dist_setup(backend: str = "nccl"):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch
        import torch.distributed as dist
        if backend == "nccl":
            torch.cuda.set_device(local)  # before NCCL init: one GPU per rank
        if not dist.is_initialized():
            dist.init_process_group(backend)
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def allmax(ws, v: float) -> float:
    """max over ranks (device tensor under NCCL, host tensor under gloo)."""
    if ws == 1:
        return v
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def weak_scaling_value(ws: int, dof_per_rank: int, local_total_ms: float, steps: int):
    """Whole-job throughput: all ranks' DoFs / max-over-ranks time (GDoF/s), and ms/step."""
    tot_ms = allmax(ws, local_total_ms)
    ms = tot_ms / steps
    return ws * dof_per_rank / (ms * 1e-3) / 1e9, ms


# ----------------------------------------------------------------------------------- GPU arm
def time_workload(cfgname: str, steps: int, warmup: int, ws: int, path: str = "auto", e2e: bool = True,
                  split: bool = True):
    import torch
    from paper_1811_06797_b200 import workloads
    cfg = synth.CONFIGS[cfgname]
    knots, w, x = synth.draw_problem(cfg)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    op = workloads.build_operator(cfg, w)
    torch.cuda.synchronize()
    setup_ms = (time.perf_counter() - t0) * 1e3
    info = op.info_dict()
    stream = torch.cuda.Stream()
    xd = torch.from_numpy(x).cuda()
    N = op.ndof
    with torch.cuda.stream(stream):
        if cfg.kkt:
            out = torch.empty_like(xd)
            run = lambda: op.kkt_apply(xd, out, cfg.n_t, cfg.tau, cfg.beta, path=path, stream=stream)
            dof = 3 * cfg.n_t * N
            flops = cfg.n_t * (op_kkt_flops(op))
        else:
            ym = torch.empty_like(xd)
            ys = torch.empty_like(xd)
            # one step = the mass part then the stiffness part (the same launches a combined
            # apply issues); the event between them times the dominant stiffness kernel (+ its
            # fixup) live inside the timed region, on the launching stream
            mid = []

            def run():
                if not split:  # one combined call (the library may overlap the two parts)
                    op.apply(xd, ym, ys, path=path, stream=stream)
                    return
                op.apply(xd, ym, None, path=path, stream=stream)
                if mid:
                    mid[-1].record(stream)
                op.apply(xd, None, ys, path=path, stream=stream)
            dof = cfg.batch * N
            flops = cfg.batch * info["plan_flops_per_vec"]
    for _ in range(warmup):
        run()
    stream.synchronize()
    barrier(ws)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    evm = [torch.cuda.Event(enable_timing=True) for _ in range(steps)] if (split and not cfg.kkt) else []
    with ClockSampler(torch.cuda.current_device()) as cs:
        for i in range(steps):
            ev[i][0].record(stream)
            if evm:
                mid.append(evm[i])
            run()
            ev[i][1].record(stream)
        stream.synchronize()
    torch.cuda.synchronize()
    barrier(ws)
    per = [a.elapsed_time(b) for a, b in ev]
    dom_ms = (sum(m.elapsed_time(b) for m, (_, b) in zip(evm, ev)) / steps) if evm else None
    tot_ms = sum(per)
    tot_ms = allmax(ws, tot_ms)
    ms = tot_ms / steps
    res = {"cfg": cfg, "op": op, "info": info, "ms": ms, "min_ms": min(per), "dof": dof, "flops": flops, "dom_ms": dom_ms,
           "setup_ms": setup_ms, "clocks": cs.summary(), "x": x, "stream": stream}
    if e2e and not cfg.kkt:
        # end to end through the public host API: pinned host buffers, H2D + apply + D2H per step
        xh = torch.from_numpy(x).pin_memory()
        ymh = torch.empty_like(xh).pin_memory()
        ysh = torch.empty_like(xh).pin_memory()
        xn, ymn, ysn = xh.numpy(), ymh.numpy(), ysh.numpy()
        op.apply_host(xn, ymn, ysn, path=path, stream=stream)
        barrier(ws)
        t0 = time.perf_counter()
        k = max(1, min(steps, 5))
        for _ in range(k):
            op.apply_host(xn, ymn, ysn, path=path, stream=stream)
        e2e_s = allmax(ws, (time.perf_counter() - t0) / k)
        res["e2e"] = {"value": ws * dof / e2e_s / 1e9, "unit": "GDoF/s", "h2d_bytes_per_step": int(x.nbytes),
                      "d2h_bytes_per_step": int(2 * x.nbytes)}
    elif e2e and cfg.kkt:
        xh = torch.from_numpy(x).pin_memory()
        oh = torch.empty_like(xh).pin_memory()
        op.kkt_apply_host(xh.numpy(), oh.numpy(), cfg.n_t, cfg.tau, cfg.beta, path=path, stream=stream)
        t0 = time.perf_counter()
        k = max(1, min(steps, 5))
        for _ in range(k):
            op.kkt_apply_host(xh.numpy(), oh.numpy(), cfg.n_t, cfg.tau, cfg.beta, path=path, stream=stream)
        e2e_s = allmax(ws, (time.perf_counter() - t0) / k)
        res["e2e"] = {"value": ws * dof / e2e_s / 1e9, "unit": "GDoF/s", "h2d_bytes_per_step": int(x.nbytes),
                      "d2h_bytes_per_step": int(x.nbytes)}
    return res


def op_kkt_flops(op) -> float:
    """Algorithmic flops of one KKT time step: 3 mass applies + 2 stiffness applies (43R plan)."""
    i = op.info_dict()
    return i["plan_flops_mass"] * 3 + i["plan_flops_stiff"] * 2 if "plan_flops_mass" in i else 0.0


def launches_per_step(info: dict, path: str, kkt: bool) -> int:
    """Our kernels per step: fused v2 = (k_canon + k_fixup) per part; KKT = k_kkt_combos + one mass
    launch over 3 n_t vectors + two accumulating stiffness launches (each with its fixup)."""
    if info.get("fused2_ok") and path != "unfused":
        return 1 + 2 * 2 if kkt else 4
    if info["fused_ok"] and path != "unfused":
        return 4 if kkt else 1
    r = info["n_rounds"]
    return (1 + 3 * 3 * r) if kkt else 3 * r


def time_dominant_kernel(res):
    """The dominant kernel of the step is the stiffness k_canon (+ its boundary fixup): its time is
    the CUDA-event interval from the end of the mass part to the end of the step, measured on the
    launching stream inside the timed region (time_workload); algorithmic flops = plan flops of the
    stiffness part x batch."""
    cfg = res["cfg"]
    if cfg.kkt or res.get("dom_ms") is None:
        return None
    flops = cfg.batch * res["info"]["plan_flops_stiff"]
    return {"kernel": "k_canon<ShapeStiffA> + k_fixup4 (stiffness part)", "ms": res["dom_ms"], "flops": flops}


def measured_traffic(workload: str):
    """dram__bytes_read+write per launch of the dominant kernel from the committed ncu --set full
    capture (profiles/traffic.json), or None."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        return t.get(workload)
    except Exception:
        return None


# ----------------------------------------------------------------------------------- CPU arm
class OracleSample:
    """The CPU oracle on a bounded sample of a workload, the way SURVEY §8(d) times it: the rows of
    `planes` z-planes of the full-size matrices are assembled by tensor Gauss quadrature
    (oracle.assemble_csr_rows; assembly timed separately) and applied by the oracle's naive CSR
    SpMV to the workload's own input vector.  A c4 (KKT) step is the paper's three rows per time
    step on those spatial rows: 3 mass + 2 stiffness SpMVs (oracle.kkt_apply's work per step)."""

    def __init__(self, cfgname: str, planes: int = 1):
        import oracle
        self.oracle = oracle
        self.cfg = cfg = synth.CONFIGS[cfgname]
        knots, w, x = synth.draw_problem(cfg)
        self.P = P = oracle.problem_from_config(cfg, w)
        N = P.ndof
        mx, my, mz = P.dims
        z0 = mz // 2
        self.r0, self.r1 = z0 * mx * my, min(mz, z0 + planes) * mx * my
        oracle.set_threads(0)
        t0 = time.perf_counter()
        self.M, self.S = oracle.assemble_csr_rows(P, self.r0, self.r1)
        self.assembly_s = time.perf_counter() - t0
        self.x = np.ascontiguousarray(x.reshape(-1, N)[0])
        self.rows = self.r1 - self.r0
        # DoFs one step processes: rows x (1 for the apply's M and S outputs; 3 blocks for a KKT step)
        self.dof = self.rows * (3 if cfg.kkt else 1)
        self.sample = ("rows [%d, %d) (%d z-planes) of the full-size %s matrices (CSR, %d nnz per matrix), "
                       "one input vector" % (self.r0, self.r1, planes, cfg.name, self.M.nnz))

    def step(self):
        sp = self.oracle.spmv
        if self.cfg.kkt:
            for _ in range(3):
                sp(self.M, self.x)
            for _ in range(2):
                sp(self.S, self.x)
        else:
            sp(self.M, self.x)
            sp(self.S, self.x)

    def rate(self, threads: int, reps: int = 3) -> float:
        """GDoF/s at `threads` OpenMP threads (0 = all cores): median of `reps` after 1 warm-up."""
        self.oracle.set_threads(threads)
        self.step()
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            self.step()
            ts.append(time.perf_counter() - t0)
        self.oracle.set_threads(0)
        return self.dof / statistics.median(ts) / 1e9


def cpu_baseline(cfgname: str, matfree: bool = True):
    """cpu_baseline of the JSON line: oracle CSR SpMV at all cores (value) and at
    1 thread, assembly time separately; plus (c3) the matrix-free element-loop route on one full
    vector at all cores."""
    cores = len(os.sched_getaffinity(0))
    s = OracleSample(cfgname)
    v_all = s.rate(0)
    v_one = s.rate(1)
    out = {"value": v_all, "unit": "GDoF/s", "cores": cores, "kind": "oracle", "route": "csr_spmv",
           "sample": s.sample, "value_1thread": v_one, "assembly_s_sample": s.assembly_s,
           "assembly_rows_per_s": s.rows / s.assembly_s}
    if matfree and not s.cfg.kkt and s.P.ndof <= 4 * 1024 * 1024:
        t0 = time.perf_counter()
        s.oracle.apply_matfree(s.P, s.x.reshape(1, *s.x.shape))
        out["matfree_value"] = s.P.ndof / (time.perf_counter() - t0) / 1e9
        out["matfree_sample"] = "one full %s vector, element loop, all cores" % s.cfg.name
    return out


def time_kkt_solve(rtol: float = 1e-8):
    """NEXT-1: all-at-once c4 KKT solve (preconditioned MINRES, iga_kkt_minres) for a tracking
    right-hand side [tau M yhat; 0; 0]; wall time of the call (it synchronises per iteration)."""
    import torch
    import synth
    from paper_1811_06797_b200 import workloads
    cfg = synth.CONFIGS["c4"]
    op = workloads.build_operator(cfg, synth.draw_weights(cfg))
    m = cfg.n - 2
    g = torch.Generator(device="cuda").manual_seed(7)
    yhat = torch.randn((cfg.n_t, m, m, m), dtype=torch.float64, device="cuda", generator=g)
    b = torch.zeros((3, cfg.n_t, m, m, m), dtype=torch.float64, device="cuda")
    ym = torch.empty_like(yhat)
    op.apply(yhat, ym, None)
    b[0] = cfg.tau * ym
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    prec = op.kkt_preconditioner(cfg.n_t, cfg.tau, cfg.beta)
    t1 = time.perf_counter()
    x = torch.empty_like(b)
    info = op.kkt_minres(b, x, cfg.n_t, cfg.tau, cfg.beta, rtol=rtol, maxit=3000, prec=prec)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    ax = torch.empty_like(b)
    op.kkt_apply(x, ax, cfg.n_t, cfg.tau, cfg.beta)
    rel2 = float(torch.linalg.vector_norm(b - ax) / torch.linalg.vector_norm(b))
    unk = 3 * cfg.n_t * m ** 3
    return {"workload": "c4_kkt_solve_pminres", "unknowns": unk, "rtol_Pinv_norm": rtol, "iters": info.iters,
            "converged": bool(info.converged), "solve_s": t2 - t1, "ms_per_iter": 1e3 * (t2 - t1) / max(info.iters, 1),
            "prec_setup_s": t1 - t0, "rel_residual_2norm": rel2}


def time_tt(ranks=(20, 20), reps: int = 50):
    """NEXT-3: the reduced-system matvec of Block AMEn (Eq. (KKT_red)) on the c4 operator:
    interfaces of the middle site (y) for TT cores of ranks (R1, R2), then
    y = sum_t c_t (L_t (x) K_t^y (x) R_t) x on a local core [R1][m][R2] (stiffness, the largest
    term set), and one A v of a TT vector; CUDA-event times on one stream."""
    import torch
    from paper_1811_06797_b200 import workloads
    cfg = synth.CONFIGS["c4"]
    op = workloads.build_operator(cfg, synth.draw_weights(cfg))
    mx, my, mz = op.dims
    R1, R2 = ranks
    g = torch.Generator(device="cuda").manual_seed(3)
    gz = torch.randn((mz, R1), dtype=torch.float64, device="cuda", generator=g)
    gy = torch.randn((R1, my, R2), dtype=torch.float64, device="cuda", generator=g)
    gx = torch.randn((R2, mx), dtype=torch.float64, device="cuda", generator=g)
    T = len(op.terms(1)[1])
    L = torch.empty((T, R1, R1), dtype=torch.float64, device="cuda")
    R = torch.empty((T, R2, R2), dtype=torch.float64, device="cuda")
    x = torch.randn((R1, my, R2), dtype=torch.float64, device="cuda", generator=g)
    y = torch.empty_like(x)
    wz = torch.empty((T, mz, R1), dtype=torch.float64, device="cuda")
    wy = torch.empty((T, R1, my, R2), dtype=torch.float64, device="cuda")
    wx = torch.empty((T, R2, mx), dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream()

    def timed(fn):
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps):
            fn()
        e1.record(s)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps
    t_if = timed(lambda: op.tt_interfaces(1, 1, gz, gy, gx, L, R))
    t_loc = timed(lambda: op.tt_local_apply(1, 1, L, R, x, y))
    t_kron = timed(lambda: op.tt_kron_apply(1, gz, gy, gx, wz, wy, wx))
    p = op.info_dict()["p"][1]
    flops_loc = 2.0 * T * R1 * my * R2 * (R2 + (2 * p + 1) + R1)
    return {"workload": "c4_tt_local_apply (Block-AMEn reduced matvec, site y)", "terms": T, "ranks": [R1, R2],
            "local_unknowns": R1 * my * R2, "interfaces_ms": t_if, "local_apply_ms": t_loc,
            "local_apply_gflops": flops_loc / (t_loc * 1e-3) / 1e9, "tt_kron_apply_ms": t_kron}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="c3")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--path", default="auto", choices=["auto", "fused", "unfused"])
    ap.add_argument("--no-extra", action="store_true", help="skip the other configs")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    a = ap.parse_args()
    warmup = max(3, a.warmup)

    if a.impl == "reference":
        ws = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        if rank != 0:
            return
        # the CPU oracle on the host cores: each step = the CSR SpMVs of a bounded sample (one
        # z-plane of rows) of the same workload; assembly of the sample runs once, untimed
        cores = len(os.sched_getaffinity(0))
        s = OracleSample(a.config)
        for _ in range(warmup):
            s.step()
        t0 = time.perf_counter()
        for _ in range(a.steps):
            s.step()
        el = time.perf_counter() - t0
        val = s.dof * a.steps / el / 1e9
        cfg = synth.CONFIGS[a.config]
        line = {"metric": "GDoF/s of fp64 low-rank Kronecker operator/KKT apply; % of roofline",
                "impl": "reference", "value": val, "unit": "GDoF/s", "n_gpus": a.gpus, "steps": a.steps,
                "warmup": warmup, "ms_per_step": 1e3 * el / a.steps, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": cfg.name, "global_batch": cfg.batch},
                "cpu_baseline": {"value": val, "unit": "GDoF/s", "cores": cores, "kind": "oracle",
                                 "route": "csr_spmv", "sample": s.sample, "assembly_s_sample": s.assembly_s},
                "e2e": {"value": val, "unit": "GDoF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    ws, rank, local = dist_setup()
    import torch
    torch.cuda.set_device(local)
    from paper_1811_06797_b200 import workloads  # noqa: F401  (fails loudly without the .so)
    res = time_workload(a.config, a.steps, warmup, ws, path=a.path)
    cfg = res["cfg"]
    ms = res["ms"]
    value = ws * res["dof"] / (ms * 1e-3) / 1e9
    achieved_step = res["flops"] / (ms * 1e-3) / 1e12
    peak = PEAK_FP64_TFLOPS
    dom = time_dominant_kernel(res)
    if dom:
        achieved = dom["flops"] / (dom["ms"] * 1e-3) / 1e12
    else:
        achieved = achieved_step
    launches = launches_per_step(res["info"], a.path, cfg.kkt)
    line = {
        "metric": "GDoF/s of fp64 low-rank Kronecker operator/KKT apply; % of roofline",
        "value": value, "unit": "GDoF/s", "n_gpus": ws, "steps": a.steps, "warmup": warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded N(0,1) inputs, seeded separable sine weights; DESIGN.md §3)",
        "config": {"workload": cfg.name, "n": cfg.n, "p": cfg.p, "R": cfg.R, "batch_per_gpu": cfg.batch,
                   "global_batch": cfg.batch * ws, "parallelism": "dp%d (batch sharded, no collective)" % ws,
                   "path": a.path, "l2": "inputs (%.0f MB) larger than L2 (126 MB); no flush" % (res["x"].nbytes / 1e6)},
        "roofline": {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": measured_traffic(cfg.name),
                     "kernel": dom["kernel"] if dom else "whole step",
                     "kernel_ms": dom["ms"] if dom else ms,
                     "step_achieved": achieved_step, "step_frac": achieved_step / peak,
                     "note": "FP64 DFMA pipe (bound 'alu'); peak = measured DFMA/DMMA rate 37.0 TF/s "
                             "(tools/ubench.cu, profiles/r01_ubench.md; nominal 37.2 at 1965 MHz). achieved = "
                             "algorithmic flops (2*nnz per banded mode product, DESIGN.md 5.2) of the dominant "
                             "kernel / its CUDA-event time inside the timed region (mass part -> end of step, "
                             "launching stream); step_* = whole mass+stiffness step. traffic = "
                             "ncu dram bytes per launch (profiles/traffic.json)"},
        "gpu_launches": launches * a.steps,
        "clocks": res["clocks"],
        "setup_ms": res["setup_ms"],
        "plan": {k: res["info"][k] for k in ("n_rounds", "n_xprod", "n_yprod", "n_zprod", "plan_flops_per_vec",
                                              "fused_ok")},
    }
    if "e2e" in res:
        line["e2e"] = res["e2e"]
    if rank == 0 and ws == 1 and not a.no_extra:
        extra = {}
        for other in ("c2", "c5", "c4"):
            if other == a.config:
                continue
            try:
                r2 = time_workload(other, max(3, min(a.steps // 2, 50)), 3, 1, path=a.path, e2e=False, split=False)
                v2 = r2["dof"] / (r2["ms"] * 1e-3) / 1e9
                ach = r2["flops"] / (r2["ms"] * 1e-3) / 1e12 if r2["flops"] else None
                extra[other] = {"workload": r2["cfg"].name, "GDoF_s": v2, "ms": r2["ms"],
                                "tflops": ach, "frac": (ach / peak) if ach else None}
                del r2
                torch.cuda.empty_cache()
            except Exception as e:  # report, never hide
                extra[other] = {"error": repr(e)}
        try:
            extra["tt"] = time_tt()
        except Exception as e:  # report, never hide
            extra["tt"] = {"error": repr(e)}
        try:
            extra["c4_solve"] = time_kkt_solve()
        except Exception as e:  # report, never hide
            extra["c4_solve"] = {"error": repr(e)}
        line["configs"] = extra
    if rank == 0 and ws == 1 and not a.no_cpu:
        line["cpu_baseline"] = cpu_baseline(a.config)
    if rank == 0:
        print(json.dumps(line))
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
