"""Executed SASS instructions of one kernel in an ncu report, grouped into runs of equal
execution count (basic blocks), largest first:
  python tools/ncu_blocks.py REP KERNEL_REGEX [MIN_MILLION_INSTR]"""
import collections
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
floor = float(sys.argv[3]) if len(sys.argv) > 3 else 0.5
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass', '--kernel-name',
                      f'regex:{kern}'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
ai, si, ei = h.index('Address'), h.index('Source'), h.index('Instructions Executed')
seen, blocks, cur = set(), [], None
for r in rows[2:]:
    try:
        e = int(r[ei])
    except (ValueError, IndexError):
        continue
    if r[ai] in seen:  # the page lists the kernel's code once per view
        continue
    seen.add(r[ai])
    toks = r[si].split()
    op = (toks[1] if toks and toks[0].startswith('@') else toks[0]).split('.')[0] if toks else '?'
    if cur is None or cur[0] != e:
        cur = [e, collections.Counter(), r[ai]]
        blocks.append(cur)
    cur[1][op] += 1
tot = sum(e * sum(c.values()) for e, c, _ in blocks)
print(f'total {tot / 1e6:.1f}M warp instructions')
for e, c, a in sorted(blocks, key=lambda b: -b[0] * sum(b[1].values())):
    n = sum(c.values())
    if e * n >= floor * 1e6:
        print(f'{a[-5:]} exec {e:8d} x {n:4d} = {e * n / 1e6:6.1f}M  {dict(c.most_common(7))}')
