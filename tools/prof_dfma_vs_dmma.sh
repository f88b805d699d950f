#!/bin/bash
# ncu --set full of the DMMA analysis and of the DFMA analysis (SWSDC_ANA_DFMA=1), config 1
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --soak 0 --no-cpu-baseline --no-mlsdc"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none -k regex:"ana_kernel" -s 2 -c 1 -o gpurun_out/prof_dmma $CMD > gpurun_out/ncu_dmma.log 2>&1 && \
SWSDC_ANA_DFMA=1 ncu --set full --clock-control none -k regex:"ana_dfma_kernel" -s 2 -c 1 -o gpurun_out/prof_dfma $CMD > gpurun_out/ncu_dfma.log 2>&1
echo "rc=$?"
