"""Per-instance key metrics of every kernel in an ncu report (grid size distinguishes
the fine / coarse launches of one step)."""
import csv, subprocess, sys
rep = sys.argv[1]
want = ['Duration', 'Grid Size', 'Registers Per Thread', 'Achieved Occupancy', 'Theoretical Occupancy',
        'Issue Slots Busy', 'L2 Hit Rate', 'DRAM Throughput', 'Compute (SM) Throughput']
out = subprocess.run(['ncu', '-i', rep, '--page', 'details', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
ii, ki, mi, vi, ui = h.index('ID'), h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('Metric Unit')
seen = {}
for r in rows[1:]:
    if r[mi] in want:
        seen.setdefault((int(r[ii]), r[ki][:50]), {})[r[mi]] = r[vi] + ' ' + r[ui]
for (i, k), d in sorted(seen.items()):
    print(i, k)
    for m in want:
        if m in d:
            print(f"    {m:28s} {d[m]}")
