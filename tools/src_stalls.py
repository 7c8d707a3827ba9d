"""Aggregate an `ncu --page source --csv --print-source sass` export by address range:
stall samples per region (hot loop vs. the rest), top stalled instructions."""
import csv
import sys
from collections import Counter, defaultdict

path = sys.argv[1]
rows = list(csv.reader(open(path)))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
base = int(data[0]["Address"], 16)
stall_cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
tot = Counter()
regions = defaultdict(Counter)
cuts = [int(x, 16) for x in sys.argv[2:]]  # region boundaries as kernel-relative offsets
per_ins = []
for d in data:
    off = int(d["Address"], 16) - base
    reg = sum(1 for c in cuts if off >= c)
    s = {c: int(d[c] or 0) for c in stall_cols}
    n = int(d["Warp Stall Sampling (All Samples)"] or 0)
    ex = int(d["Instructions Executed"] or 0)
    regions[reg]["samples"] += n
    regions[reg]["inst"] += ex
    for c, v in s.items():
        regions[reg][c] += v
        tot[c] += v
    per_ins.append((n, hex(off), d["Source"].strip()[:70], max(s, key=s.get) if n else "", ex))
T = sum(regions[r]["samples"] for r in regions)
print("total samples", T)
for r in sorted(regions):
    R = regions[r]
    top = sorted(((v, c) for c, v in R.items() if c.startswith("stall_")), reverse=True)[:6]
    print("region %d: samples %.1f%% inst %d  " % (r, 100 * R["samples"] / max(T, 1), R["inst"]),
          ", ".join("%s %.1f%%" % (c[6:], 100 * v / max(T, 1)) for v, c in top))
print("\ntop instructions:")
for n, off, src, st, ex in sorted(per_ins, reverse=True)[:40]:
    print("%6d %8s %-70s %-16s %d" % (n, off, src, st, ex))
