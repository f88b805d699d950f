#!/bin/bash
# ncu --set full of kernels matching regex $2 inside one graph step of MLSDC config $1
# ($3 = launch count, $4 = report name)
mkdir -p gpurun_out
python tools/one_step.py $1 > gpurun_out/plain_step_$1.log 2>&1 && \
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "step/" \
    -k regex:"$2" -c ${3:-1} -o gpurun_out/${4:-prof_step} $(echo python tools/one_step.py $1) > gpurun_out/ncu_${4:-prof_step}.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/ncu_${4:-prof_step}.log
