"""Aggregate executed instructions / stall samples of k_render_rays by phase.

  python scripts/phase_profile.py <cubin> <kernel-substr> <ncu_sass.csv> <render_kernel.cuh>
The phase of an instruction = the innermost RayWorker method / helper (by line
range in render_kernel.cuh) in its inline chain."""
import csv
import re
import subprocess
import sys
from collections import Counter


def ranges(src):
    lines = open(src).read().splitlines()
    marks = []
    for i, l in enumerate(lines, 1):
        m = re.match(r"\s*(?:template <[^>]*>\s*)?(?:__device__|__global__)[^(]*?(\w+)\(", l)
        if m:
            marks.append((i, m.group(1)))
    return marks


def phase_of(line, marks):
    name = "?"
    for i, n in marks:
        if i <= line:
            name = n
    return name


def main():
    cubin, kern, csvp, src = sys.argv[1:5]
    marks = ranges(src)
    txt = subprocess.run(["nvdisasm", "--print-line-info-inline", cubin], capture_output=True,
                         text=True).stdout.splitlines()
    i0 = next(i for i, l in enumerate(txt) if l.startswith(".text.") and kern in l)
    chain, off2ph, fresh = [], {}, True
    for l in txt[i0 + 1:]:
        if l.strip().startswith(".section") and off2ph:
            break
        m = re.search(r'//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?', l)
        if m:
            if fresh:
                chain, fresh = [], False
            chain.append((m.group(1).split("/")[-1], int(m.group(2))))
            if m.group(3):
                chain.append((m.group(3).split("/")[-1], int(m.group(4))))
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
        if m:
            fresh = True
            rk = [c for c in chain if c[0] == "render_kernel.cuh"]
            other = [c for c in chain if c[0] in ("quantize.cuh", "device_math.cuh")]
            ph = phase_of(rk[0][1], marks) if rk else "?"
            if other and ph in ("insert_hits",):
                ph = "quantize(" + other[0][0] + ")"
            off2ph[int(m.group(1), 16)] = ph
    if csvp == "-":  # static code size only
        code = Counter(off2ph.values())
        for ph, v in code.most_common():
            print(f"{ph:28s} {v:6d}")
        print(f"{'total':28s} {sum(code.values()):6d}")
        return
    rows = list(csv.reader(open(csvp)))
    hdr = rows[1]
    I = {h: i for i, h in enumerate(hdr)}
    base = None
    ex, st = Counter(), Counter()
    for r in rows[2:]:
        try:
            a = int(r[0], 16)
        except ValueError:
            continue
        base = a if base is None else base
        ph = off2ph.get(a - base, "?")
        ex[ph] += int(r[I["Instructions Executed"]])
        st[ph] += int(r[I["Warp Stall Sampling (All Samples)"]])
    te, ts = sum(ex.values()), sum(st.values())
    code = Counter(off2ph.values())
    print(f"{'phase':28s} {'exec':>11s} {'stall':>13s} {'SASS instrs':>12s}")
    for ph, v in ex.most_common():
        print(f"{ph:28s} exec {v / te * 100:5.1f}%   stall {st[ph] / ts * 100:5.1f}%   {code[ph]:6d}")
    print(f"{'total':28s} {'':11s} {'':13s}   {sum(code.values()):6d}")


if __name__ == "__main__":
    main()
