# usage: ab_env.sh VAR "v0 v1" -> config-1 stages + config-2 step for each value, twice
VAR=$1; VALS=$2
for rep in 1 2; do for v in $VALS; do
  echo "$VAR=$v"; env $VAR=$v bash tools/stages_cfg1.sh; env $VAR=$v python tools/one_step.py config2 | head -1
done; done
