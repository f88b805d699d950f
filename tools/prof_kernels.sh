#!/bin/bash
# ncu --set full of the four transform kernels on the config-1 bench (1 GPU).
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --soak 0 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k regex:"syn_kernel|ana_kernel|f2g_kernel|g2f_kernel" -s 4 -c 4 \
    -o gpurun_out/prof_k $CMD > gpurun_out/ncu_full.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/ncu_full.log
