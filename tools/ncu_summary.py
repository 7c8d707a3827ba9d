"""Summarise an ncu --set full report (raw page) into markdown for profiles/."""
import csv
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active % (of peak)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__inst_executed_pipe_lsu.sum.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__inst_executed_pipe_tmem.sum.pct_of_peak_sustained_active", "TMEM pipe %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "DFMA thread-instructions"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("sm__warps_active.avg.per_cycle_active", "warps active / SM"),
]
STALLS = ["wait", "short_scoreboard", "long_scoreboard", "math_pipe_throttle", "not_selected", "selected",
          "no_instruction", "mio_throttle", "barrier", "branch_resolving", "dispatch_stall"]


def main(rep, title):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    print("# %s\n" % title)
    print("Report: `%s` (ncu --set full --clock-control none; cold, serialised replay)\n" % rep)
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        print("## %s\n" % d.get("Kernel Name", "?")[:120])
        print("| metric | value |\n|---|---|")
        for k, name in KEYS:
            if k in d:
                print("| %s | %s %s |" % (name, d[k], u.get(k, "")))
        for k in hdr:  # FP64 tensor-core (DMMA) pipe counters, where the report has them
            if "dmma" in k and (k.endswith("pct_of_peak_sustained_active") or k.endswith(".sum")):
                print("| %s | %s %s |" % (k, d[k], u.get(k, "")))
        print("\nStall reasons (warp cycles per issued instruction):\n")
        print("| stall | per issue |\n|---|---|")
        for s in STALLS:
            k = "smsp__average_warps_issue_stalled_%s_per_issue_active.ratio" % s
            if k in d:
                print("| %s | %s |" % (s, d[k]))
        print()


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "ncu summary")
