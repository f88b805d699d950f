"""Summarise an ncu report (details + stall reasons) for the profiles/ notes."""
import csv
import subprocess
import sys

rep = sys.argv[1]
want = ['Duration', 'DRAM Throughput', 'Compute (SM) Throughput', 'Achieved Occupancy',
        'Theoretical Occupancy', 'Registers Per Thread', 'Block Size', 'Grid Size',
        'Dynamic Shared Memory Per Block', 'Executed Ipc Active', 'Issue Slots Busy',
        'Eligible Warps Per Scheduler', 'Active Warps Per Scheduler', 'L1/TEX Hit Rate', 'L2 Hit Rate']
out = subprocess.run(['ncu', '-i', rep, '--page', 'details', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
ki, mi, vi, ui = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('Metric Unit')
seen = {}
for r in rows[1:]:
    if r[mi] in want:
        seen.setdefault(r[ki][:40], {})[r[mi]] = r[vi] + ' ' + r[ui]
for k, d in seen.items():
    print(k)
    for m in want:
        if m in d:
            print('   ', m.ljust(36), d[m])
raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h = rows[0]
names = [r[h.index('Kernel Name')][:24] for r in rows[2:]]
keys = ['sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_bytes.sum']
print('stalls / pipes:', names)
for i, col in enumerate(h):
    if col in keys or ('pcsamp_warps_issue_stalled' in col and not col.endswith('not_issued')):
        try:
            vals = [float(r[i].replace(',', '')) for r in rows[2:]]
        except ValueError:
            continue
        unit = rows[1][i]
        # ncu picks byte units per metric; report bytes in MB so columns compare
        scale = {'byte': 1e-6, 'Kbyte': 1e-3, 'Mbyte': 1.0, 'Gbyte': 1e3}.get(unit)
        if scale is not None:
            vals = [v * scale for v in vals]
            unit = 'MB'
        if max(vals) > 0.5 or col in keys:
            print('  ', (col[-52:] + f' [{unit}]').ljust(60), ' '.join(f'{v:11.2f}' for v in vals))
