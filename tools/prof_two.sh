#!/bin/bash
# ncu --set full of the two Fourier kernels on the config-1 bench.
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --soak 0 --no-cpu-baseline --no-mlsdc"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k regex:"f2g|g2f" -s 2 -c 2 -o gpurun_out/prof_two $CMD > gpurun_out/ncu_two.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/ncu_two.log
