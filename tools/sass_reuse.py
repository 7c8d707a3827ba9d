"""Static SASS check of the FP64 register-operand economics of a kernel's hottest loop.

On sm_100a a DFMA whose three 64-bit source operands all come from the register file (no
operand-reuse-cache hit, not RZ) issues at 3 cycles instead of 2 (tools/ubench_rf.cu:
25.6 vs 31-33 TF/s).  This script finds the backward-branch loop with the most FP64
instructions in `cuobjdump -sass` output and reports how many of them read 3 fresh operands,
plus a static-issue estimate of the loop's FP64 pipe ceiling.
usage: python tools/sass_reuse.py <file.o|.so> <mangled-name-substring>
"""
import re
import subprocess
import sys
from collections import Counter


def parse(text):
    lines = text.splitlines()
    ins = []
    i = 0
    while i < len(lines):
        m = re.match(r'\s+/\*([0-9a-f]{4,})\*/\s+(.*?);\s+/\* (0x[0-9a-f]+) \*/', lines[i])
        if m:
            hi = int(re.search(r'/\* (0x[0-9a-f]+) \*/', lines[i + 1]).group(1), 16)
            t = m.group(2).strip()
            ins.append((int(m.group(1), 16), t, (hi >> 41) & 0xf))
            i += 2
        else:
            i += 1
    return ins


def is_fp(t):
    op = t.split()[1] if t.startswith('@') else t.split()[0]
    return op.split('.')[0] in ('DFMA', 'DMUL', 'DADD')


def fresh_counts(body):
    """Per FP64 instruction: register source operands not served by the operand-reuse cache.
    Model: an instruction that reads operand slot i replaces that slot's cached register (kept
    only if the operand carries .reuse); slots it does not read keep their cached register."""
    c = Counter()
    cache = {}
    for a, t, s in body:
        if t.startswith('@'):
            t = t.split(None, 1)[1]
        parts = t.split(None, 1)
        if len(parts) < 2:
            continue
        srcs = [o.strip() for o in parts[1].split(',')][1:]
        f = 0
        for i, s_ in enumerate(srcs):
            r = s_.replace('.reuse', '')
            isreg = r.startswith('R') and r != 'RZ' and re.match(r'R\d+$', r)
            if isreg and cache.get(i) == r and is_fp(t):
                pass
            elif isreg and is_fp(t):
                f += 1
            if isreg or r.startswith('['):
                cache[i] = r if s_.endswith('.reuse') else None
        if is_fp(t):
            c[f] += 1
    return c


def main():
    path, name = sys.argv[1], sys.argv[2]
    out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    funcs = re.split(r'\n\s+Function : ', out)
    for f in funcs[1:]:
        fname = f.split('\n', 1)[0].strip()
        if name not in fname:
            continue
        ins = parse(f)
        best = None
        for a, t, s in ins:
            m = re.search(r'BRA(?:\.\S+)?\s+(?:!?U?P\w+,\s*)?(0x[0-9a-f]+)', t)
            if m and int(m.group(1), 16) < a:
                lo = int(m.group(1), 16)
                body = [x for x in ins if lo <= x[0] <= a]
                nfp = sum(1 for x in body if is_fp(x[1]))
                if best is None or nfp > best[0]:
                    best = (nfp, lo, a, body)
        nfp, lo, hi, body = best
        c = fresh_counts(body)
        cyc = sum(3 if k >= 3 else 2 for k in c.elements())
        stall = sum(s for _, _, s in body)
        print("%s\n  loop %#x-%#x: %d instr, %d FP64, fresh-operand histogram %s, 3-fresh %.1f%%, "
              "pipe cycles %d (%.2f/FP64), static stall sum %d" %
              (fname[:110], lo, hi, len(body), nfp, dict(sorted(c.items())), 100.0 * c[3] / max(nfp, 1), cyc,
               cyc / max(nfp, 1), stall))


if __name__ == "__main__":
    main()
