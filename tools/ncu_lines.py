"""Stall samples per CUDA source line for one kernel of an ncu report (needs -lineinfo)."""
import csv
import subprocess
import sys
from collections import defaultdict

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '-k', 'regex:' + kern,
                      '--print-source', 'cuda,sass'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
fname, agg, text = None, defaultdict(int), {}
hdr = None
for r in rows:
    if len(r) == 2 and r[0] == 'File Path':
        fname = r[1].split('/')[-1]
        continue
    if r and r[0] == 'Line No':
        hdr = r
        si = hdr.index('Warp Stall Sampling (All Samples)')
        continue
    if hdr is None or len(r) != len(hdr) or not r[0].isdigit():
        continue
    key = (fname, int(r[0]))
    text[key] = r[1].strip()[:90]
    try:
        agg[key] += int(r[si] or 0)
    except ValueError:
        pass
tot = sum(agg.values())
print('total samples', tot)
for key, v in sorted(agg.items(), key=lambda kv: -kv[1])[:n]:
    print(f"{v:6d} {100 * v / max(tot, 1):5.1f}%  {key[0]}:{key[1]:<5d} {text[key]}")
