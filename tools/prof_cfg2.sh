#!/bin/bash
# ncu --set full of the config-2 F_E kernels in one graph step; text summaries only
mkdir -p gpurun_out
python tools/one_step.py config2 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "step/" \
    -k regex:"syn_kernel|ana_kernel|swe_grid5|sweep_node|finalize" -c 12 \
    -o /tmp/r02_cfg2 python tools/one_step.py config2 > gpurun_out/r02_cfg2_ncu.log 2>&1
echo "rc=$?"
python tools/ncu_instances.py /tmp/r02_cfg2.ncu-rep > gpurun_out/r02_cfg2_instances.txt 2>&1
for k in syn_kernel ana_kernel swe_grid5 sweep_node finalize; do
  python tools/ncu_lines.py /tmp/r02_cfg2.ncu-rep $k 16 > gpurun_out/r02_cfg2_lines_$k.txt 2>&1
done
