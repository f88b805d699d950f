#!/bin/bash
for cfg in "SWSDC_ANA_LSPLIT=1" "SWSDC_ANA_LSPLIT=2" "SWSDC_ANA_TMA=2"; do
  echo -n "$cfg "
  env $cfg python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-mlsdc --soak 0.3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['stages_ms_per_launch']['legendre_analysis'])"
done
