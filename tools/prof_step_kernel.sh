#!/bin/bash
# ncu --set full of one kernel (regex $2) inside one graph step of MLSDC config $1
mkdir -p gpurun_out
python tools/one_step.py $1 > gpurun_out/plain_step.log 2>&1 && \
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "step/" \
    -k regex:"$2" -c ${3:-1} -o gpurun_out/prof_step $(echo python tools/one_step.py $1) > gpurun_out/ncu_step.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/ncu_step.log
