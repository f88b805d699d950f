#!/bin/bash
# Evidence for profiles/: bench line, ncu launch list (timing shares), ncu --set full of
# the transform kernels and of the fused F_E kernels (config 2 step).  1 GPU.
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
CMD="python bench.py --steps 2 --warmup 3 --soak 0 --no-cpu-baseline --no-mlsdc"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k regex:"syn_kernel|ana_kernel|f2g_kernel|g2f_kernel" -s 4 -c 4 \
    -o gpurun_out/prof_k $CMD > gpurun_out/ncu_full.log 2>&1
CMD2="python tools/stage_profile.py config2"
$CMD2 > gpurun_out/stage_cfg2.log 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k regex:"swe_grid_kernel|sweep_node|spec_combine|finalize_swe" -s 12 -c 4 \
    -o gpurun_out/prof_swe $CMD2 > gpurun_out/ncu_swe.log 2>&1
echo "rc=$?"
