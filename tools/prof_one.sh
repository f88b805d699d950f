#!/bin/bash
# ncu --set full of one kernel (regex $1) on the config-1 bench, launch skip $2.
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --soak 0 --no-cpu-baseline --no-mlsdc"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k regex:"$1" -s ${2:-2} -c 1 -o gpurun_out/prof_one $CMD > gpurun_out/ncu_one.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/ncu_one.log
