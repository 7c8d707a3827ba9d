"""Split an `ncu --page source --csv --print-source sass` export of one kernel into regions:
the FP64 sweep (first to last hot FP64 instruction), the code before it (segment/round setup,
barriers, coefficient loads) and after it (plane retire, flush), and report each region's share
of the warp-stall samples and of the executed FP64 instructions, its FP64-pipe activity estimate,
plus the top stall reasons and the most-sampled instructions.
usage: python tools/stall_regions.py <export.csv> [SM count] [clock MHz] [kernel ms]"""
import csv
import sys
from collections import Counter


def main(path, sms=148, mhz=1965.0, ms=None):
    rows = list(csv.reader(open(path)))
    # an export can repeat the kernel block: keep the first one
    nxt = [i for i, r in enumerate(rows) if i > 0 and r and r[0] == "Kernel Name"]
    if nxt:
        rows = rows[:nxt[0]]
    title = rows[0][1] if len(rows[0]) > 1 else "?"
    hdr = rows[1]
    data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr) and r[0] != "Address"]
    base = int(data[0]["Address"], 16)
    stall_cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
    ins = []
    for d in data:
        src = d["Source"].strip()
        op = (src.split()[1] if src.startswith("@") and len(src.split()) > 1 else (src.split()[0] if src else ""))
        ex = int(d["Instructions Executed"] or 0)
        ins.append((int(d["Address"], 16) - base, src, op.startswith(("DFMA", "DMUL", "DADD")), ex,
                    int(d["Warp Stall Sampling (All Samples)"] or 0), {c: int(d[c] or 0) for c in stall_cols}))
    hot = max(ex for _, _, fp, ex, _, _ in ins if fp)
    fpa = [a for a, _, fp, ex, _, _ in ins if fp and ex >= hot / 4]
    lo, hi = min(fpa), max(fpa)
    regs = {"before sweep (setup, round start, coefficient loads)": lambda a: a < lo,
            "sweep (X/Y/Z stages)": lambda a: lo <= a <= hi,
            "after sweep (plane retire, flush)": lambda a: a > hi}
    T = sum(x[4] for x in ins)
    F = sum(x[3] for x in ins if x[2])
    print("# Stall-sample regions: %s\n" % title[:140])
    print("Source: `%s` (ncu --set full --import-source on, SASS source page)\n" % path)
    print("| region | samples | FP64 instr | top stalls (share of all samples) |\n|---|---|---|---|")
    for name, f in regs.items():
        sel = [x for x in ins if f(x[0])]
        smp = sum(x[4] for x in sel)
        fp = sum(x[3] for x in sel if x[2])
        st = Counter()
        for x in sel:
            st.update(x[5])
        top = ", ".join("%s %.1f%%" % (k[6:], 100.0 * v / T) for k, v in st.most_common(4) if v)
        print("| %s | %.1f %% | %.1f %% | %s |" % (name, 100.0 * smp / T, 100.0 * fp / F, top))
    if ms:
        sweep_share = sum(x[4] for x in ins if lo <= x[0] <= hi) / T
        fp_sweep = sum(x[3] for x in ins if x[2] and lo <= x[0] <= hi)
        cyc = ms * 1e-3 * mhz * 1e6 * sms * 4 * sweep_share
        print("\nFP64-pipe activity inside the sweep ≈ %.1f %% (2 SMSP-cycles per warp FP64 op over the sweep's "
              "share of %.3f ms)" % (100.0 * 2 * fp_sweep / cyc, ms))
    print("\nMost-sampled instructions:\n\n| offset | instruction | samples | top stall |\n|---|---|---|---|")
    for x in sorted(ins, key=lambda x: -x[4])[:12]:
        top = max(x[5], key=x[5].get)
        print("| %#x | `%s` | %.2f %% | %s |" % (x[0], x[1][:60], 100.0 * x[4] / T, top[6:]))


if __name__ == "__main__":
    a = sys.argv
    main(a[1], int(a[2]) if len(a) > 2 else 148, float(a[3]) if len(a) > 3 else 1965.0, float(a[4]) if len(a) > 4 else None)
