"""Atomic-throughput counters of the splat / move kernels from an ncu report captured
with tools/prof_round2.sh (the --metrics list there):
  python tools/ncu_atomics.py report.ncu-rep"""
import csv
import subprocess
import sys

WANT = [
    ("gpu__time_duration.sum", "duration (ns)"),
    ("smsp__inst_executed_op_global_red.sum", "RED instructions executed (warp-level)"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_red.sum", "L1 global RED requests"),
    ("l1tex__m_l1tex2xbar_write_sectors_mem_global_op_red.sum", "L1->L2 RED sectors"),
    ("lts__t_requests_srcunit_tex_op_red.sum", "L2 RED requests (from SMs)"),
    ("lts__t_sectors_srcunit_tex_op_red.sum", "L2 RED sectors (from SMs)"),
    ("lts__t_sectors_srcunit_tex_op_red_lookup_hit.sum", "L2 RED sector hits"),
    ("lts__t_sectors_srcunit_tex_op_red_lookup_miss.sum", "L2 RED sector misses"),
    ("lts__t_sectors_op_red.sum", "L2 RED sectors (all units)"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput (% of peak)"),
    ("dram__bytes_read.sum", "DRAM read bytes"),
    ("dram__bytes_write.sum", "DRAM write bytes"),
]


def main(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    k = hdr.index("Kernel Name")
    for r in data:
        name = r[k].split("(")[0]
        if not any(x in name for x in ("splat", "sample", "place_points", "unpermute")):
            continue
        print(f"--- {name}")
        vals = {}
        for m, label in WANT:
            if m in hdr:
                v = r[hdr.index(m)]
                vals[m] = v
                print(f"    {label:42s} {v:>16s} {units[hdr.index(m)]}")
        try:
            t = float(vals["gpu__time_duration.sum"].replace(",", "")) * 1e-9
            req = float(vals["lts__t_requests_srcunit_tex_op_red.sum"].replace(",", ""))
            print(f"    {'L2 RED request rate':42s} {req / t / 1e9:16.1f} G/s")
        except (KeyError, ValueError, ZeroDivisionError):
            pass


if __name__ == "__main__":
    main(sys.argv[1])
