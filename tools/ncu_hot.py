"""Top SASS lines by stall samples for one kernel in an ncu report (source page)."""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--kernel-name', f'regex:{kern}'],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
si = hdr.index('Warp Stall Sampling (All Samples)'); src = hdr.index('Source'); ex = hdr.index('Instructions Executed')
data = []
for r in rows[2:]:
    try:
        data.append((int(r[si]), r[src].strip(), int(r[ex]), r[0]))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
print('total samples', tot, 'instructions', sum(d[2] for d in data))
for smp, s, e, a in sorted(data, reverse=True)[:top]:
    print(f'{smp / tot:6.3f} {e:9d} {a[-5:]} {s[:90]}')
