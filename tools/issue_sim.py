"""Toy in-order issue model of one SM sub-partition running W warps through the same SASS
loop body: FP64 pipe accepts one warp instruction per 2 cycles, results ready 8 cycles after
issue (DFMA/DMUL/DADD), LDS results after ~30, one instruction issued per cycle.  Used to
ask whether a Legendre inner loop's FP64-pipe shortfall is explained by its dependency
structure alone.

    python tools/issue_sim.py tools/leg_pattern_probe.bin a2m_patternILi4ELi8ELi3ELi0 [--warps 4]
"""
import argparse
import re
import subprocess

LAT = {"DFMA": 8, "DMUL": 8, "DADD": 8, "LDS": 30, "LDG": 400, "SHFL": 20}
FP64 = {"DFMA", "DMUL", "DADD"}


def regs(tok, width):
    m = re.match(r"-?\|?R(\d+)", tok.strip())
    if not m or tok.strip().startswith("RZ"):
        return []
    b = int(m.group(1))
    return list(range(b, b + width))


def parse(sass_text):
    ins = []
    for line in sass_text.splitlines():
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    return ins


def loop_body(ins):
    """largest backward-branch loop body that contains FP64 work"""
    best = None
    for a, t in ins:
        m = re.search(r"BRA.*?(0x[0-9a-f]+)", t)
        if m and int(m.group(1), 16) < a:
            lo = int(m.group(1), 16)
            body = [tt for ad, tt in ins if lo <= ad <= a]
            n = sum(1 for tt in body if tt.split()[0].split(".")[0] in FP64)
            if n and (best is None or n > best[0]):
                best = (n, body)
    return best[1]


def decode(body):
    out = []
    for t in body:
        if t.startswith("@"):
            t = t.split(None, 1)[1]
        parts = t.split(None, 1)
        op = parts[0]
        base = op.split(".")[0]
        ops = [o.strip() for o in parts[1].split(",")] if len(parts) > 1 else []
        w = 2 if base in FP64 else 1
        if base == "LDS":
            w = 4 if ".128" in op else (2 if ".64" in op else 1)
        dst, src = [], []
        if base in FP64 or base in ("LDS", "IMAD", "IADD3", "MOV", "LOP3", "SHFL", "VIADD", "LEA"):
            if ops:
                dst = regs(ops[0], w)
                for o in ops[1:]:
                    o2 = o.strip("[]").split("+")[0]
                    src += regs(o2, 2 if base in FP64 else 1)
        elif base in ("STS",):
            for o in ops:
                src += regs(o.strip("[]").split("+")[0], 4 if ".128" in op else 2)
        out.append((base, dst, src))
    return out


def simulate(prog, warps, iters=60):
    ready = [dict() for _ in range(warps)]
    pc = [0] * warps
    done = [0] * warps
    fp_free = 0
    cyc = 0
    fp_issued = 0
    last = 0
    total = len(prog) * iters
    while min(done) < total:
        issued = False
        for k in range(warps):
            w = (last + 1 + k) % warps
            if done[w] >= total:
                continue
            base, dst, src = prog[pc[w]]
            if any(ready[w].get(r, 0) > cyc for r in src + dst):
                continue
            if base in FP64 and fp_free > cyc:
                continue
            for r in dst:
                ready[w][r] = cyc + LAT.get(base, 4)
            if base in FP64:
                fp_free = cyc + 2
                fp_issued += 1
            pc[w] = (pc[w] + 1) % len(prog)
            done[w] += 1
            last = w
            issued = True
            break
        cyc += 1
    return fp_issued * 2 / cyc


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("binary")
    ap.add_argument("func")
    ap.add_argument("--warps", type=int, nargs="+", default=[1, 2, 3, 4, 6])
    a = ap.parse_args()
    txt = subprocess.run(["cuobjdump", "-sass", a.binary], capture_output=True, text=True).stdout
    blocks = txt.split("Function : ")
    body = None
    for b in blocks:
        if b.startswith(("_Z", "_ZN")) and a.func in b.split("\n")[0]:
            body = loop_body(parse(b))
            break
    prog = decode(body)
    nfp = sum(1 for p in prog if p[0] in FP64)
    print(f"loop body: {len(prog)} instructions, {nfp} FP64")
    for w in a.warps:
        print(f"  {w} warps: FP64 pipe busy {100 * simulate(prog, w):.1f}%")


if __name__ == "__main__":
    main()
