#!/bin/bash
# Bench + ncu evidence for config 1 (run under gpurun from the repo root).
set -x
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
cat gpurun_out/bench.json
CMD="python bench.py --steps 2 --warmup 3 --soak 0 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k regex:"syn_kernel|ana_kernel|f2g_kernel|g2f_kernel" -s 4 -c 4 \
    -o gpurun_out/prof_cfg1 $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"
tail -5 gpurun_out/ncu_full.log
