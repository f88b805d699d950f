for rep in 1 2; do for v in old new; do
  echo "LIB=$v"; SWSDC_LIB=$PWD/abtest/lib_$v.so python tools/stage_profile.py config2 config4 2>&1 | grep -E "==|swe_grid"
done; done
