for rep in 1 2; do for v in 0 1; do
  echo "SHORT=$v"; SWSDC_ANA_SHORT=$v bash tools/stages_cfg1.sh; SWSDC_ANA_SHORT=$v python tools/one_step.py config2 | head -1
done; done
