"""SASS instructions (and optionally ncu executed-instruction / stall counts)
per source line of one kernel: nvdisasm --print-line-info output + optional
ncu source-page CSV (--print-source sass) of the same build.

  python scripts/sass_lines.py <cubin> <kernel-substring> [ncu_sass.csv]
"""
import csv
import re
import subprocess
import sys
from collections import Counter, defaultdict


def main():
    cubin, kern = sys.argv[1], sys.argv[2]
    txt = subprocess.run(["nvdisasm", "--print-line-info-inline", cubin], capture_output=True,
                         text=True).stdout.splitlines()
    own = ("render_kernel.cuh", "quantize.cuh", "device_math.cuh", "render.cu")
    i0 = next(i for i, l in enumerate(txt) if l.startswith(".text.") and kern in l)
    cur, off2line, static = None, {}, Counter()
    chain, fresh = [], True
    for l in txt[i0 + 1:]:
        if l.startswith(".text.") or l.strip().startswith(".section"):
            if off2line:
                break
        m = re.search(r'//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?', l)
        if m:
            if fresh:
                chain, fresh = [], False
            chain.append((m.group(1).split("/")[-1], int(m.group(2))))
            if m.group(3):
                chain.append((m.group(3).split("/")[-1], int(m.group(4))))
            mine = [c for c in chain if c[0] in own]
            if mine:
                inner = mine[0]
                caller = next((c for c in mine[1:] if c != inner), None)
                cur = (inner[0], inner[1] if caller is None else f"{inner[1]}<{caller[0][:6]}:{caller[1]}")
            else:
                cur = chain[0]
            continue
        if re.search(r"/\*[0-9a-f]{4,}\*/", l):
            fresh = True
        m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(\S+)", l)
        if m and cur:
            off = int(m.group(1), 16)
            off2line[off] = cur
            static[cur] += 1
    dyn, stall = Counter(), Counter()
    if len(sys.argv) > 3:
        rows = list(csv.reader(open(sys.argv[3])))
        hdr = rows[1]
        I = {h: i for i, h in enumerate(hdr)}
        base = None
        for r in rows[2:]:
            try:
                a = int(r[0], 16)
            except ValueError:
                continue
            base = a if base is None else base
            ln = off2line.get(a - base)
            if ln:
                dyn[ln] += int(r[I["Instructions Executed"]])
                stall[ln] += int(r[I["Warp Stall Sampling (All Samples)"]])
    tot_s, tot_d, tot_st = sum(static.values()), sum(dyn.values()) or 1, sum(stall.values()) or 1
    print(f"static SASS instructions: {tot_s}")
    key = dyn if dyn else static
    for ln, _ in key.most_common(45):
        print(f"{ln[0]}:{str(ln[1]):>18s}  static {static[ln]:5d}  exec {dyn[ln]/tot_d*100:5.1f}%  stall {stall[ln]/tot_st*100:5.1f}%")


if __name__ == "__main__":
    main()
