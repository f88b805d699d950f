#!/bin/bash
# Same-box A/B of the committed tree (abtest/old, a worktree with its own build)
# against the working tree: MLSDC graph steps and config-1 stages.
for rep in 1 2; do
  for t in abtest/old .; do
    echo "TREE=$t"
    (cd $t && for c in ${CFGS:-config2 config0 config4}; do python tools/one_step.py $c | head -1; done)
  done
done
