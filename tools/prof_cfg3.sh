#!/bin/bash
# ncu --set full of the config-3 (T1279) F_E kernels in one graph step; text summaries only
mkdir -p gpurun_out
python tools/one_step.py config3 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "step/" \
    -k regex:"syn_kernel|ana_kernel|swe_prod" -c 6 \
    -o /tmp/r02_cfg3 python tools/one_step.py config3 > gpurun_out/r02_cfg3_ncu.log 2>&1
echo "rc=$?"
python tools/ncu_summary.py /tmp/r02_cfg3.ncu-rep > gpurun_out/r02_cfg3_ncu_summary.txt 2>&1
for k in ana_kernel syn_kernel swe_prod; do
  python tools/ncu_lines.py /tmp/r02_cfg3.ncu-rep $k 20 > gpurun_out/r02_cfg3_lines_$k.txt 2>&1
done
ncu -i /tmp/r02_cfg3.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum,lts__t_bytes.sum > gpurun_out/r02_cfg3_traffic.csv 2>&1
