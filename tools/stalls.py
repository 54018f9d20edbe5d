"""Warp-stall breakdown of an ncu capture (reads the report here, no GPU needed).

    python tools/stalls.py gpurun_out/c4_leg2.ncu-rep map2alm [--top 30] [--range A B]

Prints the per-reason stall shares, the hottest 50-instruction SASS regions and the top
instructions by samples (with their dominant stall reasons).
"""
import argparse
import collections
import csv
import io
import subprocess

COLS = ["stall_long_sb", "stall_wait", "stall_math", "stall_short_sb", "stall_not_selected",
        "stall_selected", "stall_no_inst", "stall_branch_resolving", "stall_dispatch", "stall_mio",
        "stall_lg", "stall_barrier", "stall_membar"]


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("kernel")
    ap.add_argument("--top", type=int, default=30)
    ap.add_argument("--range", type=int, nargs=2)
    ap.add_argument("--skip", type=int, default=0, help="launches of the matching kernels to skip")
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "sass",
                          "--kernel-name", "regex:" + a.kernel,
                          "--launch-skip", str(a.skip), "--launch-count", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    data = []
    for r in rows[2:]:  # first captured launch only
        if r and r[0] == "Kernel Name":
            break
        if len(r) == len(h):
            data.append(r)
    si = h.index("Warp Stall Sampling (All Samples)")
    ei = h.index("Instructions Executed")
    ci = {c: h.index(c) for c in COLS if c in h}
    tot = sum(f(r[si]) for r in data)
    print(f"{len(data)} SASS lines, {tot:.0f} samples")
    sums = {c: sum(f(r[j]) for r in data) for c, j in ci.items()}
    for c, v in sorted(sums.items(), key=lambda kv: -kv[1]):
        if v / tot > 0.005:
            print(f"  {c[6:]:18s} {100 * v / tot:5.1f}%")
    b = collections.defaultdict(float)
    for i, r in enumerate(data):
        b[i // 50] += f(r[si])
    print("hot regions:", " ".join(f"{k * 50}:{100 * v / tot:.1f}%" for k, v in sorted(b.items()) if v / tot > 0.01))
    idx = range(*a.range) if a.range else sorted(sorted(range(len(data)), key=lambda i: -f(data[i][si]))[: a.top])
    for i in idx:
        r = data[i]
        why = " ".join(f"{c[6:10]}={r[j]}" for c, j in ci.items() if f(r[j]) > 0.002 * tot)
        print(f"{i:5d} {r[1][:56]:56s} {r[ei]:>10s} {100 * f(r[si]) / tot:5.2f}% {why}")


if __name__ == "__main__":
    main()
