#!/bin/bash
# Same-box A/B of library builds abtest/lib_<v>.so for v in ${LIBS:-old new}:
# graph step of each MLSDC config in ${CFGS}, plus config-1 stages if STAGES=1; alternated REPS times.
for rep in $(seq ${REPS:-2}); do for v in ${LIBS:-old new}; do
  for c in ${CFGS:-config2 config4}; do
    echo "LIB=$v $(SWSDC_LIB=$PWD/abtest/lib_$v.so python tools/one_step.py $c | head -1)"
  done
  if [ "${STAGES:-0}" = 1 ]; then echo "LIB=$v"; SWSDC_LIB=$PWD/abtest/lib_$v.so bash tools/stages_cfg1.sh; fi
done; done
