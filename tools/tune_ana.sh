#!/bin/bash
# analysis us/launch at config 1 for each forced latitude split and the automatic choice
for cfg in "SWSDC_ANA_LSPLIT=1" "SWSDC_ANA_LSPLIT=2" "SWSDC_ANA_LSPLIT=3" "SWSDC_ANA_LSPLIT=4" "SWSDC_AUTO=1"; do
  echo -n "$cfg "
  env $cfg python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-mlsdc --soak 0.3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['stages_ms_per_launch']['legendre_analysis']*1e3, 1))"
done
