#!/bin/bash
# Per-kernel time breakdown (ncu launch list, cold caches off) of one graph step of each MLSDC config
mkdir -p gpurun_out
for cfg in ${@:-config2 config0 config4}; do
  python tools/one_step.py $cfg | head -1
  ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --cache-control none \
      --clock-control none --csv --log-file gpurun_out/brk_$cfg.csv python tools/one_step.py $cfg > /dev/null 2>&1
  python - $cfg <<'PY'
import csv, sys, re
from collections import defaultdict
cfg = sys.argv[1]
rows = [r for r in csv.reader(open(f"gpurun_out/brk_{cfg}.csv")) if len(r) > 5]
h = rows[0]; vi = h.index("Metric Value"); ni = h.index("Kernel Name")
agg = defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    k = re.sub(r"\(.*", "", r[ni]).replace("void ", "").replace("(anonymous namespace)::", "")
    t = float(r[vi].replace(",", ""))
    agg[k][0] += 1; agg[k][1] += t
tot = sum(v[1] for v in agg.values())
print(f"{cfg}: {sum(v[0] for v in agg.values())} kernels, sum {tot/1e3:.1f} us")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"  {k[:60]:60s} {n:4d} {t/1e3:9.1f} us {t/n/1e3:7.2f} us/launch {100*t/tot:5.1f}%")
PY
done
