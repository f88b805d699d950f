#!/bin/bash
# sum of per-kernel durations of one graph step vs the step's wall time
for cfg in ${@:-config2 config0}; do
  python tools/one_step.py $cfg
  ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --cache-control none \
      --clock-control none --csv --log-file gpurun_out/gap_$cfg.csv python tools/one_step.py $cfg > /dev/null 2>&1
  python - $cfg <<'PY'
import csv, sys
cfg = sys.argv[1]
rows = [r for r in csv.reader(open(f"gpurun_out/gap_{cfg}.csv")) if len(r) > 5]
h = rows[0]; vi = h.index("Metric Value"); ni = h.index("Kernel Name")
ts = [float(r[vi].replace(",", "")) for r in rows[1:]]
unit = rows[1][h.index("Metric Unit")]
print(cfg, "kernels", len(ts), "sum", round(sum(ts), 1), unit)
PY
done
