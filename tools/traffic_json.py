"""profiles/traffic_<workload>.json from an ncu launch list (gpu__time_duration.sum,
dram__bytes_read.sum, dram__bytes_write.sum):  per-launch DRAM bytes of each kernel of
the iteration, averaged over its launches.
python tools/traffic_json.py LAUNCHES.csv WORKLOAD [source-command]"""
import csv
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from bench import NCU_NAMES  # noqa: E402

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, mi, vi, ii = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('ID')
launches = {}
for r in rows[1:]:
    launches.setdefault(int(r[ii]), {'k': r[ki]})[r[mi]] = float(r[vi].replace(',', ''))
agg = {}
# the C2 iteration scans its chains with chains_reg_kernel; a chains_kernel in the same
# list then belongs to the integral API calls bench.py makes at 4096^2
reg = any('chains_reg_kernel' in x['k'] for x in launches.values())
for x in launches.values():
    full = x['k'].replace('void ', '').replace('inim::', '')
    base = full.split('<')[0].split('(')[0]
    name = NCU_NAMES.get(base)
    if base == 'write_kernel' and full.split('>')[0].endswith(', 0'):
        name = 'write_tables'  # the integral API's tables mode, not the iteration's field
    if base == 'chains_kernel' and reg:
        name = 'chains_integral'
    if name is None:
        continue
    a = agg.setdefault(name, [0, 0.0, 0.0])
    a[0] += 1
    a[1] += x.get('dram__bytes_read.sum', 0.0) + x.get('dram__bytes_write.sum', 0.0)
    a[2] += x.get('gpu__time_duration.sum', 0.0)
out = {"workload": sys.argv[2], "source": sys.argv[3] if len(sys.argv) > 3 else sys.argv[1],
       "per_launch_bytes": {k: int(v[1] / v[0]) for k, v in agg.items()},
       "per_launch_us_cold": {k: round(v[2] / v[0] / 1e3, 2) for k, v in agg.items()},
       "launches": {k: v[0] for k, v in agg.items()}}
dst = Path(__file__).resolve().parent.parent / "profiles" / f"traffic_{sys.argv[2]}.json"
dst.write_text(json.dumps(out, indent=1) + "\n")
print(dst, json.dumps(out["per_launch_bytes"]))
