"""Summarise ncu captures (gpurun_out/*.ncu-rep, launches.csv) into profiles/ (committed).

    python tools/summarize_profiles.py <round-tag>

Writes profiles/<tag>_launches.md (per-kernel share of the bench command's launch list),
profiles/<tag>_ncu.md (per-kernel key metrics of the full captures, incl. the ncu-executed
DP FLOP rate 2*DFMA + DMUL + DADD over the kernel time) and profiles/ncu_kernels.json (DRAM
bytes per launch of each captured kernel; bench.py reads it for roofline.traffic).
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "gpurun_out"
PROF = ROOT / "profiles"

METRICS = [
    "gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum.per_cycle_elapsed",
    "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum.per_cycle_elapsed",
    "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum.per_cycle_elapsed", "smsp__cycles_elapsed.avg",
    "smsp__cycles_active.avg",
]


def short(name):
    name = name.replace("shtk::", "")
    name = name.split("(")[0].replace("void ", "")
    if name.startswith("ring_p2"):  # size classes share a kernel name: keep <M, E, MINB, BLUE>
        return name.replace(" ", "")
    return name.split("<")[0]


def raw_rows(rep):
    r = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True)
    rows = list(csv.reader(io.StringIO(r.stdout)))
    h = rows[0]
    units = rows[1]
    return h, units, rows[2:]


def to_float(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return float("nan")


def kernel_table(rep):
    h, units, rows = raw_rows(rep)
    out = []
    for v in rows:
        d = {"kernel": short(v[h.index("Kernel Name")])}
        for m in METRICS:
            if m in h:
                d[m] = to_float(v[h.index(m)])
                d[m + ".unit"] = units[h.index(m)]
        t = d["gpu__time_duration.sum"]
        tu = d["gpu__time_duration.sum.unit"]
        t_s = t * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}.get(tu, 1e-9)
        cyc = d.get("smsp__cycles_elapsed.avg", 0)
        dp = cyc * (2 * d.get("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum.per_cycle_elapsed", 0) +
                    d.get("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum.per_cycle_elapsed", 0) +
                    d.get("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum.per_cycle_elapsed", 0))
        d["executed_dp_flop"] = dp
        d["time_s"] = t_s
        d["executed_dp_tflops"] = dp / t_s / 1e12 if t_s > 0 else float("nan")
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd = d.get("dram__bytes_read.sum", 0) * mult.get(d.get("dram__bytes_read.sum.unit", "byte"), 1)
        wr = d.get("dram__bytes_write.sum", 0) * mult.get(d.get("dram__bytes_write.sum.unit", "byte"), 1)
        d["dram_bytes"] = rd + wr
        d["clock_mhz"] = d.get("smsp__cycles_active.avg", 0) / t_s / 1e6 if t_s > 0 else float("nan")
        out.append(d)
    return out


def launches(csvfile):
    tot = defaultdict(float)
    cnt = defaultdict(int)
    with open(csvfile) as f:
        lines = [l for l in f if l.startswith('"')]
    rd = csv.reader(lines)
    h = next(rd)
    for v in rd:
        if v[h.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        k = short(v[h.index("Kernel Name")])
        unit = v[h.index("Metric Unit")]
        val = to_float(v[h.index("Metric Value")]) * {"ns": 1e-9, "us": 1e-6, "ms": 1e-3}.get(unit, 1e-9)
        tot[k] += val
        cnt[k] += 1
    return tot, cnt


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    PROF.mkdir(exist_ok=True)
    md = [f"# {tag}: ncu summaries (B200, sm_100a)\n",
          "Full captures: `ncu --set full --clock-control none` of one launch per kernel of "
          "`tools/profile_run.py --nside 2048 --lmax 4096` (C4). Executed DP rate = "
          "(2*DFMA + DMUL + DADD thread instructions) / kernel time; the algorithmic rate "
          "(bench.py roofline) counts 8 flops per reference pair-step over the same time.\n"]
    traffic = {}
    for rep in sorted(OUT.glob("c4_*.ncu-rep")):
        rows = kernel_table(rep)
        md.append(f"\n## {rep.name}\n")
        md.append("| kernel | grid x block | regs | time ms | clock MHz | warps active % | FP64 pipe % | issue % | "
                  "DRAM MB | DRAM % | executed DP TFLOP/s |")
        md.append("|---|---|---|---|---|---|---|---|---|---|---|")
        for d in rows:
            md.append("| {k} | {g:.0f} x {b:.0f} | {r:.0f} | {t:.3f} | {c:.0f} | {w:.1f} | {f:.1f} | {i:.1f} | {dm:.1f} | {dp:.1f} | {tf:.2f} |".format(
                k=d["kernel"], g=d.get("launch__grid_size", 0), b=d.get("launch__block_size", 0),
                r=d.get("launch__registers_per_thread", 0), t=d["time_s"] * 1e3, c=d["clock_mhz"],
                w=d.get("sm__warps_active.avg.pct_of_peak_sustained_active", 0),
                f=d.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 0),
                i=d.get("smsp__issue_active.avg.pct_of_peak_sustained_active", 0),
                dm=d["dram_bytes"] / 1e6, dp=d.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 0),
                tf=d["executed_dp_tflops"]))
            traffic.setdefault(d["kernel"], {
                "dram_bytes": d["dram_bytes"], "time_ms": d["time_s"] * 1e3,
                "executed_dp_tflops": d["executed_dp_tflops"],
                "fp64_pipe_pct": d.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 0),
                "source": f"profiles/{tag}_ncu.md ({rep.name})"})
    (PROF / f"{tag}_ncu.md").write_text("\n".join(md) + "\n")
    (PROF / "ncu_kernels.json").write_text(json.dumps(traffic, indent=1) + "\n")
    lf = OUT / "launches.csv"
    if lf.exists():
        tot, cnt = launches(lf)
        s = sum(tot.values())
        lines = [f"# {tag}: launch list of `bench.py --steps 2 --warmup 3` (ncu gpu__time_duration, "
                 "cold-cache, serialised: compare shares, not absolutes)\n",
                 "| kernel | launches | total ms | share |", "|---|---|---|---|"]
        for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
            lines.append(f"| {k} | {cnt[k]} | {v * 1e3:.3f} | {100 * v / s:.1f}% |")
        (PROF / f"{tag}_launches.md").write_text("\n".join(lines) + "\n")
    bj = OUT / "bench.json"
    if bj.exists() and bj.read_text().strip():
        (PROF / f"{tag}_bench.json").write_text(bj.read_text().strip().splitlines()[-1] + "\n")
    print("wrote", sorted(p.name for p in PROF.iterdir()))


if __name__ == "__main__":
    main()
