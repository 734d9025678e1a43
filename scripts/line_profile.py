"""Executed warp instructions and stall samples per source line of a kernel.

  python scripts/line_profile.py <cubin> <kernel-substr> <ncu_sass.csv> [top]
(ncu_sass.csv: `ncu -i rep --page source --csv --print-source sass`)."""
import csv
import re
import subprocess
import sys
from collections import Counter


def main():
    cubin, kern, csvp = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    txt = subprocess.run(["nvdisasm", "--print-line-info-inline", cubin], capture_output=True,
                         text=True).stdout.splitlines()
    i0 = next(i for i, l in enumerate(txt) if l.startswith(".text.") and kern in l)
    off2line, cur, fresh = {}, None, True
    for l in txt[i0 + 1:]:
        if l.strip().startswith(".section") and off2line:
            break
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            if fresh:
                cur, fresh = (m.group(1).split("/")[-1], int(m.group(2))), False
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
        if m:
            fresh = True
            off2line[int(m.group(1), 16)] = cur
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
        if base is None:
            base = a
        ln = off2line.get(a - base)
        ex[ln] += float(r[I["Instructions Executed"]] or 0)
        st[ln] += float(r[I["Warp Stall Sampling (All Samples)"]] or 0)
    te, ts = sum(ex.values()), sum(st.values())
    print(f"{'file:line':34s} {'exec%':>7s} {'stall%':>7s}")
    for ln, v in ex.most_common(top):
        print(f"{str(ln):34s} {100 * v / te:7.2f} {100 * st[ln] / ts:7.2f}")


if __name__ == "__main__":
    main()
