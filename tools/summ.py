"""Summaries of ncu launch-list CSVs and bench JSON lines (local analysis helper)."""
import csv, collections, json, sys

def launches(p):
    rows = list(csv.reader(open(p)))
    for i, r in enumerate(rows):
        if r and r[0] == 'ID':
            hdr = r; start = i + 1; break
    agg = collections.OrderedDict()
    for r in rows[start:]:
        d = dict(zip(hdr, r))
        name = d['Kernel Name'].split('(')[0][:48]
        agg.setdefault((name, d['Metric Name']), []).append(float(d['Metric Value'].replace(',', '')))
    return agg

if __name__ == '__main__':
    for p in sys.argv[1:]:
        if p.endswith('.csv'):
            print(p)
            tot = 0
            for (name, met), vs in launches(p).items():
                avg = sum(vs) / len(vs)
                if met == 'gpu__time_duration.sum':
                    tot += sum(vs)
                print(f"  {name:48s} {met:26s} n={len(vs):3d} avg={avg:14.1f}")
            print(f"  total time (ns): {tot:.0f}")
        else:
            for line in open(p):
                if line.startswith('{'):
                    j = json.loads(line)
                    print(p, 'value', round(j['value'], 1), 'ms/step', round(j.get('ms_per_step', 0), 3), 'e2e', j.get('e2e', {}).get('value'))
                    for k, v in (j.get('kernels') or {}).items():
                        print(f"   {k:18s} {v['avg_us']:8.2f} us  x{v['launches_per_step']}  share {v['share']:.3f}")
                    print('   integral', j.get('integral_image'))
                    print('   roofline', {k: j['roofline'][k] for k in ('kernel', 'achieved', 'frac')} if j.get('roofline') else None)
