"""Regenerate _build.py's KNOWN_SPILLS ratchet from a build log (the stderr of _build.py, whose
ptxas -warn-spills lines name every spilling kernel).  Only run this after checking that the
BASELINE kernels (see the comment above KNOWN_SPILLS) do not spill.
usage: python tools/spill_ratchet.py <build.log>"""
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
log = open(sys.argv[1]).read()
ents = {}
pat = (r"function '_ZN5igalr2f27k_canonINS0_(\w+?)ELi(\d)ELi(\d+)ELi2ELi(\d)ELb1ELb1ELb([01])ELb([01])EEEvNS0_5Args2E"
       r"NS0_6KSplitE', (\d+) bytes spill stores, (\d+) bytes spill loads")
for m in re.finditer(pat, log):
    shape, P, LW, QX, sp, pk, st, ld = m.groups()
    ents[(shape, int(P), int(LW), int(QX), int(sp), int(pk))] = (int(st), int(ld))
lines = ['    _MK %% ("%s", %d, %d, %d, %d, %d): %s,' % (k + (ents[k],))
         for k in sorted(ents, key=lambda k: (k[1], k[0], k[2], k[3], k[4], k[5]))]
p = os.path.join(ROOT, "paper_1811_06797_b200", "_build.py")
s = open(p).read()
i = s.index("KNOWN_SPILLS = {")
j = s.index("}\n", i) + 2
open(p, "w").write(s[:i] + "KNOWN_SPILLS = {\n" + "\n".join(lines) + "\n}\n" + s[j:])
print("%d guarded spilling variants" % len(lines))
BASELINE = {("11ShapeStiffA", 3, 16, 4, 0, 0), ("10ShapeMassKILi4EE", 3, 16, 4, 0, 0),   # c3
            ("11ShapeStiffA", 3, 12, 2, 1, 1), ("10ShapeMassKILi4EE", 3, 12, 2, 0, 1),   # c4 (packed)
            ("11ShapeStiffA", 4, 13, 4, 0, 0), ("10ShapeMassKILi3EE", 4, 13, 4, 0, 0)}   # c5
for k in sorted(ents):
    if k in BASELINE:
        print("WARNING: a BASELINE kernel spills:", k, ents[k])
