"""Executed SASS opcode histogram of one kernel in an ncu report (source page):
  python tools/ncu_ops.py REP KERNEL_REGEX [TOP]"""
import collections
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--kernel-name', f'regex:{kern}'],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
ei, si, wi = hdr.index('Instructions Executed'), hdr.index('Source'), hdr.index('Warp Stall Sampling (All Samples)')
op, st = collections.Counter(), collections.Counter()
for r in rows[2:]:
    try:
        e = int(r[ei])
    except (ValueError, IndexError):
        continue
    w = r[si].split()
    o = (w[1] if w[0].startswith('@') else w[0]).split('.')[0]
    op[o] += e
    st[o] += int(r[wi] or 0)
tot, sst = sum(op.values()), sum(st.values()) or 1
print(f'total warp instructions {tot}, stall samples {sst}')
for o, c in op.most_common(top):
    print(f'{o:8s} {c:11d} {c / tot:6.3f}   stalls {st[o] / sst:6.3f}')
