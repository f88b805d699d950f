#!/bin/bash
for B in 3 5; do for S in 1 2 4; do
  echo -n "B=$B SPLIT=$S "
  SWSDC_SYN_B=$B SWSDC_SYN_SPLIT=$S python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-mlsdc --soak 0.3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['stages_ms_per_launch']['legendre_synthesis'])"
done; done
