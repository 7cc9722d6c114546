"""Aggregate an ncu launch list (gpu__time_duration + dram bytes per launch) per kernel:
  python tools/launch_agg.py launches.csv [--second-half]"""
import collections
import csv
import sys


def main(path, second_half):
    rows = list(csv.reader(open(path)))
    i = [k for k, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr, rows = rows[i], rows[i + 1:]
    kn, mn, mv, idc = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    per, names = collections.defaultdict(dict), {}
    for r in rows:
        per[r[idc]][r[mn]] = float(r[mv].replace(",", ""))
        names[r[idc]] = r[kn].split("(")[0]
    ids = sorted(per, key=int)
    if second_half:
        ids = ids[len(ids) // 2:]
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for i in ids:
        a, p = agg[names[i]], per[i]
        a[0] += 1
        a[1] += p.get("gpu__time_duration.sum", 0)
        a[2] += p.get("dram__bytes_read.sum", 0)
        a[3] += p.get("dram__bytes_write.sum", 0)
    tot = sum(a[1] for a in agg.values())
    print(f"{'kernel':42s} {'n':>4s} {'total_us':>10s} {'share':>6s} {'us/launch':>10s} {'rdMB/l':>8s} {'wrMB/l':>8s} {'GB/s':>6s}")
    for n, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{n[:42]:42s} {a[0]:4d} {a[1] / 1e3:10.1f} {a[1] / tot:6.3f} {a[1] / a[0] / 1e3:10.1f} "
              f"{a[2] / a[0] / 1e6:8.1f} {a[3] / a[0] / 1e6:8.1f} {(a[2] + a[3]) / a[1]:6.0f}")
    print(f"total {tot / 1e3:.1f} us over {len(ids)} launches")


if __name__ == "__main__":
    main(sys.argv[1], "--second-half" in sys.argv)
