"""Condensed per-kernel view of an ncu report (details page + top stall reasons)."""
import csv, subprocess, sys

WANT = ['Duration', 'DRAM Throughput', 'Memory Throughput', 'L1/TEX Hit Rate', 'L2 Hit Rate', 'Achieved Occupancy',
        'Theoretical Occupancy', 'Registers Per Thread', 'Compute (SM) Throughput', 'Block Size', 'Grid Size',
        'Dynamic Shared Memory Per Block', 'Executed Ipc Active', 'Warp Cycles Per Issued Instruction',
        'Block Limit Shared Mem', 'Block Limit Registers', 'Issue Slots Busy']


def main(rep):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'details', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    ki, mi, vi, ui, ii = (hdr.index(x) for x in ('Kernel Name', 'Metric Name', 'Metric Value', 'Metric Unit', 'ID'))
    cur = None
    for r in rows[1:]:
        if r[mi] in WANT:
            key = (r[ii], r[ki].split('(')[0][:50])
            if key != cur:
                print('---', key)
                cur = key
            print(f'    {r[mi]:36s} {r[vi]:>12s} {r[ui]}')
    raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr = rows[0]
    names = [h for h in hdr if h.startswith('smsp__average_warp_latency_issue_stalled') or
             h.startswith('smsp__pcsamp_warps_issue_stalled_')]
    stall = [h for h in hdr if h.startswith('smsp__pcsamp_warps_issue_stalled_') and not h.endswith('not_issued')]
    dram = [h for h in hdr if h in ('dram__bytes_read.sum', 'dram__bytes_write.sum')]
    kcol = hdr.index('Kernel Name')
    for r in rows[2:]:
        vals = []
        for h in stall:
            try:
                vals.append((float(r[hdr.index(h)].replace(',', '')), h.replace('smsp__pcsamp_warps_issue_stalled_', '')))
            except ValueError:
                pass
        vals.sort(reverse=True)
        tot = sum(v for v, _ in vals) or 1
        print(r[kcol].split('(')[0][:50], {h: r[hdr.index(h)] for h in dram},
              ' '.join(f'{n}:{v / tot:.2f}' for v, n in vals[:6]))


if __name__ == '__main__':
    main(sys.argv[1])
