"""Hottest SASS instructions of a kernel with their top stall reasons."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '-k', 'regex:' + kern,
                      '--print-source', 'sass'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
si, ni = hdr.index('Source'), hdr.index('Warp Stall Sampling (All Samples)')
stall_cols = [i for i, h in enumerate(hdr) if h.startswith('stall_') or 'Stall' in h and i != ni and 'Not-issued' not in h]
body = [r for r in rows[2:] if len(r) == len(hdr) and r[ni].isdigit()]
# keep the first kernel instance only
seen, uniq = set(), []
for r in body:
    if r[0] in seen:
        break
    seen.add(r[0]); uniq.append(r)
tot = sum(int(r[ni]) for r in uniq)
print('samples', tot, 'instructions', len(uniq))
top = sorted(range(len(uniq)), key=lambda i: -int(uniq[i][ni]))[:n]
for i in sorted(top):
    r = uniq[i]
    reasons = []
    for c in range(len(hdr)):
        h = hdr[c]
        if h.startswith('Warp Stall Sampling') or not r[c].replace('.', '').isdigit():
            continue
        if h.startswith('stall_') and 'Not Issued' not in h and float(r[c]) > 0:
            reasons.append((float(r[c]), h))
    reasons.sort(reverse=True)
    print(f"{i:5d} {int(r[ni]):5d} {r[si].strip()[:60]:60s} " + ", ".join(f"{h.split('(')[0].strip()[:22]}={v:.0f}" for v, h in reasons[:3]))
