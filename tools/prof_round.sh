#!/bin/bash
# Evidence for profiles/: bench line, ncu launch list (timing shares), ncu --set full of
# the four transform kernels (config 1) and of the F_E kernels of one config-2 graph step.
mkdir -p gpurun_out
if [ "$1" = "swe" ]; then
python tools/one_step.py config2 > gpurun_out/step_cfg2.log 2>&1 && \
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "step/" \
    -k regex:"swe_grid_reg_kernel|syn_kernel|ana_kernel|sweep_node" -c 4 \
    -o gpurun_out/prof_swe python tools/one_step.py config2 > gpurun_out/ncu_swe.log 2>&1
echo "rc=$?"; exit 0
fi
python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
CMD="python bench.py --steps 2 --warmup 3 --soak 0 --no-cpu-baseline --no-mlsdc"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k regex:"syn_kernel|ana_kernel|f2g_reg_kernel|g2f_reg_kernel" -s 4 -c 4 \
    -o gpurun_out/prof_k $CMD > gpurun_out/ncu_full.log 2>&1
echo "rc=$?"
