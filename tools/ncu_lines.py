"""Aggregate an ncu source page (cuda,sass view) per CUDA source line: stall samples and
executed warp instructions.  python tools/ncu_lines.py REP KERNEL_REGEX [TOP]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda,sass',
                      '--kernel-name', f'regex:{kern}'], capture_output=True, text=True).stdout
agg, fname, cur, hdr = {}, '', None, None
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == 'File Path':
        fname = r[1].split('/')[-1]
        continue
    if r[0] == 'Line No':
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0]:
        cur = (fname, r[0], r[1].strip()[:80])
    try:
        smp, ex = int(r[4] or 0), int(r[7] or 0)
    except ValueError:
        continue
    a = agg.setdefault(cur, [0, 0])
    a[0] += smp
    a[1] += ex
tot = sum(v[0] for v in agg.values()) or 1
ins = sum(v[1] for v in agg.values()) or 1
print(f'samples {tot}  warp-instructions {ins}')
for key, (smp, ex) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f'{smp / tot:6.3f} {ex / ins:6.3f}  {key[0]}:{key[1]}  {key[2]}')
