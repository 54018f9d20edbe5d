"""Per-source-line stall samples and executed FP64 instructions from an ncu source page
(cuda,sass view of a -lineinfo build):

    ncu -i rep --page source --csv --kernel-name regex:NAME --print-source cuda,sass > k.csv
    python tools/src_lines.py k.csv [min_pct]
"""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
minp = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
f = None
lines = {}
hdr = None
cur = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].rsplit("/", 1)[-1]
        continue
    if r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or len(r) < 6:
        continue
    if r[0] not in ("", "-"):
        cur = (f, int(r[0]), r[1].strip())
        continue
    # SASS rows under a source line: Line No empty
for r in rows:
    pass
# simpler: the source rows carry aggregated metrics for their SASS
agg = []
for r in rows:
    if len(r) > 8 and r[0].isdigit():
        try:
            s = int(r[4] or 0)
            e = int(r[7] or 0)
        except ValueError:
            continue
        agg.append((r[0], r[1].strip()[:80], s, e))
tot = sum(a[2] for a in agg) or 1
for ln, src, s, e in sorted(agg, key=lambda x: -x[2]):
    if 100 * s / tot < minp:
        break
    print(f"{100 * s / tot:5.1f}%  line {ln:>5}  exec {e:>10}  {src}")
