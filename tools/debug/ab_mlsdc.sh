for rep in 1 2; do for v in old new; do
  echo "LIB=$v"; for c in ${CFGS:-config4 config2}; do SWSDC_LIB=$PWD/abtest/lib_$v.so python tools/one_step.py $c | head -1; done
done; done
