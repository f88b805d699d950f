#!/bin/bash
# ncu --set full (source-level) of one config-1 kernel (regex $1), summaries written on the box
mkdir -p gpurun_out
n=${2:-one}
CMD="python bench.py --steps 2 --warmup 3 --soak 0 --no-cpu-baseline --no-mlsdc"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k regex:"$1" -s 2 -c 1 -o gpurun_out/p_$n $CMD > gpurun_out/ncu_$n.log 2>&1
python tools/ncu_summary.py gpurun_out/p_$n.ncu-rep > gpurun_out/s_$n.txt 2>&1
python tools/ncu_lines.py gpurun_out/p_$n.ncu-rep "$1" 60 > gpurun_out/l_$n.txt 2>&1
python tools/ncu_hot.py gpurun_out/p_$n.ncu-rep "$1" 60 > gpurun_out/h_$n.txt 2>&1
