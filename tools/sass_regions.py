"""Per-region view of an ncu source page (SASS): stall samples and executed FP64 warp
instructions of every innermost backward-branch loop and of the code outside loops.

    ncu -i rep.ncu-rep --page source --csv --kernel-name regex:NAME --print-source sass > k.csv
    python tools/sass_regions.py k.csv
"""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
end = next((i for i in range(2, len(rows)) if rows[i] and rows[i][0] == "Kernel Name"), len(rows))
rows = rows[:end]
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
ins = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    a = int(r[ix["Address"]], 16)
    t = r[ix["Source"]].strip()
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    e = int(r[ix["Instructions Executed"]] or 0)
    ins.append((a, t, s, e))
base = ins[0][0]
loops = []
for a, t, s, e in ins:
    m = re.search(r"BRA\s.*?(0x[0-9a-f]+)", t)
    if m:
        tgt = int(m.group(1), 16)
        if tgt > 0x100000:  # absolute
            tgt -= 0
        if tgt < a:
            loops.append((tgt, a))
# innermost: no other loop strictly inside
inner = [l for l in loops if not any(o != l and l[0] <= o[0] and o[1] <= l[1] for o in loops)]
tot_s = sum(x[2] for x in ins)
tot_fp = sum(x[3] for x in ins if re.match(r"(@\S+\s+)?D(FMA|MUL|ADD)", x[1]))
print(f"total samples {tot_s}, FP64 warp instr {tot_fp:.3e}")
covered = set()
for lo, hi in sorted(inner):
    body = [x for x in ins if lo <= x[0] <= hi]
    for x in body:
        covered.add(x[0])
    s = sum(x[2] for x in body)
    fp = sum(x[3] for x in body if re.match(r"(@\S+\s+)?D(FMA|MUL|ADD)", x[1]))
    n = len(body)
    nfp = sum(1 for x in body if re.match(r"(@\S+\s+)?D(FMA|MUL|ADD)", x[1]))
    print(f"loop {lo - base:#07x}-{hi - base:#07x} len {n:4d} fp64/iter {nfp:4d}  samples {100 * s / tot_s:5.1f}%  fp64 {100 * fp / max(tot_fp, 1):5.1f}%")
rest = [x for x in ins if x[0] not in covered]
s = sum(x[2] for x in rest)
fp = sum(x[3] for x in rest if re.match(r"(@\S+\s+)?D(FMA|MUL|ADD)", x[1]))
print(f"outside innermost loops: samples {100 * s / tot_s:5.1f}%  fp64 {100 * fp / max(tot_fp, 1):5.1f}%")
# hottest non-FP64 instructions
top = sorted(ins, key=lambda x: -x[2])[:25]
for a, t, s, e in top:
    print(f"  {a - base:#07x} {100 * s / tot_s:5.2f}%  {t[:70]}")
