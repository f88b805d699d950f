"""Top SASS lines by warp-stall samples for one kernel of an ncu report."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '-k', 'regex:' + kern,
                      '--print-source', 'sass'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
si, ai, ni = hdr.index('Source'), hdr.index('Address'), hdr.index('Warp Stall Sampling (All Samples)')
body = [r for r in rows[2:] if len(r) == len(hdr) and r[ni].isdigit()]
tot = sum(int(r[ni]) for r in body)
print('total samples', tot, 'instructions', len(body))
idx = sorted(range(len(body)), key=lambda i: -int(body[i][ni]))[:n]
for i in sorted(idx):
    r = body[i]
    print(f"{i:5d} {int(r[ni]):6d}  {r[si].strip()[:90]}")
