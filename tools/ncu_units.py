"""Per-kernel unit utilisation from an ncu report (raw page):  python tools/ncu_units.py REP"""
import csv
import subprocess
import sys

out = subprocess.run(['ncu', '-i', sys.argv[1], '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
ki = h.index('Kernel Name')
keys = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_sectors.sum',
        'l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum', 'l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum',
        'l1tex__t_requests_pipe_lsu_mem_global_op_st.sum', 'l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum',
        'l1tex__throughput.avg.pct_of_peak_sustained_active', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'smsp__inst_executed.sum', 'sm__warps_active.avg.pct_of_peak_sustained_active']
for v in rows[2:]:
    print(v[ki][:60])
    for k in keys:
        if k in h:
            print(f'   {k:60s} {v[h.index(k)]}')
    # breakdown of the lts / l1 throughput sub-metrics that are highest
    subs = [(float(v[i].replace(',', '')), n) for i, n in enumerate(h)
            if n.endswith('.avg.pct_of_peak_sustained_elapsed') and ('lts__' in n or 'l1tex__' in n)
            and v[i] not in ('', 'n/a')]
    for val, n in sorted(subs, reverse=True)[:6]:
        print(f'   * {n:58s} {val:.1f}')
