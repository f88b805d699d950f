#!/bin/bash
# Round-2 evidence bundle (run under gpurun from the repo root):
#   bench line, ncu launch list of the config-1 bench command (timing shares),
#   ncu --set full of the four config-1 transform kernels, and of the F_E
#   kernels of one config-4 graph step.  Outputs under gpurun_out/r02_<tag>_*.
TAG=${1:-v1}
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/r02_${TAG}_gputest.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/r02_${TAG}_gputest.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r02_${TAG}_bench.json 2> gpurun_out/r02_${TAG}_bench.err
echo "bench rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --soak 0 --no-cpu-baseline --no-mlsdc"
$CMD > gpurun_out/r02_${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file gpurun_out/r02_${TAG}_cfg1_launches.csv $CMD > gpurun_out/r02_${TAG}_ncu_list.log 2>&1
echo "list rc=$?"
ncu --set full --clock-control none --import-source on \
    -k regex:"syn_kernel|ana_kernel|f2g_reg_kernel|g2f_reg_kernel" -s 4 -c 4 \
    -o gpurun_out/r02_${TAG}_cfg1 $CMD > gpurun_out/r02_${TAG}_ncu_cfg1.log 2>&1
echo "full cfg1 rc=$?"
python tools/one_step.py config4 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "step/" \
    -k regex:"swe_grid5|syn_kernel|ana_kernel" -c 3 \
    -o gpurun_out/r02_${TAG}_cfg4 python tools/one_step.py config4 > gpurun_out/r02_${TAG}_ncu_cfg4.log 2>&1
echo "full cfg4 rc=$?"
bash tools/step_breakdown.sh config0 config2 config4 config3 > gpurun_out/r02_${TAG}_step_breakdowns.txt 2>&1
echo "breakdown rc=$?"
# summarise on the box, keep only text (the reports exceed gpurun's copy-back cap)
for rep in cfg1 cfg4; do
  python tools/ncu_summary.py gpurun_out/r02_${TAG}_${rep}.ncu-rep > gpurun_out/r02_${TAG}_${rep}_ncu_summary.txt 2>&1
  ncu -i gpurun_out/r02_${TAG}_${rep}.ncu-rep --page raw --csv \
      --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum > gpurun_out/r02_${TAG}_${rep}_traffic.csv 2>&1
done
for k in syn_kernel ana_kernel f2g_reg g2f_reg; do
  python tools/ncu_lines.py gpurun_out/r02_${TAG}_cfg1.ncu-rep $k 20 > gpurun_out/r02_${TAG}_cfg1_lines_$k.txt 2>&1
done
python tools/ncu_lines.py gpurun_out/r02_${TAG}_cfg4.ncu-rep swe_grid5 25 > gpurun_out/r02_${TAG}_cfg4_lines_swe_grid5.txt 2>&1
mkdir -p /tmp/reps && mv gpurun_out/*.ncu-rep /tmp/reps/ 2>/dev/null
rm -f gpurun_out/brk_*.csv
du -sh gpurun_out
