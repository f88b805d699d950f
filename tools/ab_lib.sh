#!/bin/bash
# Same-box A/B of two library builds: abtest/lib_old.so vs abtest/lib_new.so
# (config-1 stage times and value, config-2 graph step), alternated twice.
for rep in 1 2; do for v in old new; do
  echo "LIB=$v"
  SWSDC_LIB=$PWD/abtest/lib_$v.so bash tools/stages_cfg1.sh
  SWSDC_LIB=$PWD/abtest/lib_$v.so python tools/one_step.py ${CFG:-config2} | head -1
done; done
