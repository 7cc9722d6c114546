"""Summarise an ncu --csv launch list (gpu__time_duration.sum [+ dram bytes]) per kernel name.
python tools/launch_table.py launches.csv [skip_first_n_launches]"""
import csv
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
h = rows[0]
ki, mi, vi, ii = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('ID')
launches = OrderedDict()
for r in rows[1:]:
    launches.setdefault(int(r[ii]), {'k': r[ki].split('(')[0].replace('void ', '')})[r[mi]] = float(
        r[vi].replace(',', ''))
agg = OrderedDict()
for i, x in list(launches.items())[skip:]:
    a = agg.setdefault(x['k'], [0, 0.0, 0.0, 0.0])
    a[0] += 1
    a[1] += x.get('gpu__time_duration.sum', 0.0)
    a[2] += x.get('dram__bytes_read.sum', 0.0)
    a[3] += x.get('dram__bytes_write.sum', 0.0)
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':45s} {'n':>4s} {'avg_us':>8s} {'share':>6s} {'rd_MB':>8s} {'wr_MB':>8s}")
for k, (n, t, rd, wr) in agg.items():
    print(f"{k[:45]:45s} {n:4d} {t / n / 1e3:8.2f} {t / tot:6.3f} {rd / n / 1e6:8.2f} {wr / n / 1e6:8.2f}")
print(f"total {tot / 1e3:.1f} us")
