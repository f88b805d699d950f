#!/bin/bash
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --soak 0 --no-cpu-baseline --no-mlsdc"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k regex:"syn_kernel|ana_kernel|f2g_reg_kernel|g2f_reg_kernel" -s 4 -c 4 \
    -o gpurun_out/s5_cfg1 $CMD > gpurun_out/ncu_s5_cfg1.log 2>&1
ncu -i gpurun_out/s5_cfg1.ncu-rep --page raw --csv > gpurun_out/s5_cfg1_raw.csv 2>/dev/null
python tools/lsu_view.py gpurun_out/s5_cfg1_raw.csv
