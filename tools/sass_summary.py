"""Per-kernel SASS instruction counts of libinim.so (static, from cuobjdump -sass): the
evidence that the reduce stages tiles with TMA (UTMALDG), that the splats use
warp-aggregated integer reductions (MATCH + REDG / RED), that the smoothing taps are
FFMA immediates, and the register / shared-memory budget of every kernel.

  python tools/sass_summary.py [libinim.so] > profiles/round2_sass_summary.txt
"""
import re
import subprocess
import sys
from collections import Counter, defaultdict
from pathlib import Path

LIB = Path(sys.argv[1]) if len(sys.argv) > 1 else Path(__file__).resolve().parent.parent / "paper_2408_06513_b200" / "libinim.so"
KEYS = ["UTMALDG", "UBLKCP", "SYNCS", "MATCH", "REDG", "RED", "ATOMG", "ATOM", "FFMA2", "FFMA", "DFMA", "DADD", "LDG", "STG",
        "LDS", "STS", "SHFL", "BAR", "FMNMX"]


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
    return [o.split("(")[0] for o in out]


def main():
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", str(LIB)], capture_output=True, text=True).stdout
    res = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-res-usage", str(LIB)], capture_output=True, text=True).stdout
    counts = defaultdict(Counter)
    name = None
    for line in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            name = m.group(1)
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if m and name:
            op = m.group(1)
            counts[name]["total"] += 1
            for k in KEYS:
                if op == k or op.startswith(k + "."):
                    counts[name][k] += 1
            if op.startswith("FFMA") and re.search(r",\s*-?[0-9.]+e?-?\d*\s*,", line):
                counts[name]["FFMA_imm"] += 1
    regs = {}
    cur = None
    for line in res.splitlines():
        m = re.match(r"\s*Function (\S+):", line)
        if m:
            cur = m.group(1)
        m = re.search(r"REG:(\d+) STACK:(\d+) SHARED:(\d+)", line)
        if m and cur:
            regs[cur] = m.groups()
            cur = None
    names = sorted(counts)
    pretty = dict(zip(names, demangle(names)))
    print(f"# static SASS instruction counts per kernel of {LIB.name} (sm_100a); REG/STACK/SHARED from -res-usage")
    cols = ["total"] + KEYS + ["FFMA_imm"]
    print("kernel | REG STACK SHARED | " + " ".join(cols))
    for n in sorted(names, key=lambda x: pretty[x]):
        c = counts[n]
        r = regs.get(n, ("?", "?", "?"))
        vals = " ".join(f"{k}={c[k]}" for k in cols if c[k])
        print(f"{pretty[n]} | {r[0]} {r[1]} {r[2]} | {vals}")


if __name__ == "__main__":
    main()
