#!/bin/bash
# ncu evidence for profiles/: launch lists (gpu__time_duration) + one --set full per top kernel
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for w in motion720 motion720gray motion4k dpd1 dpd3 dpd5; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$w.csv \
     python bench.py --workload $w --steps 2 --warmup 3 --no-cpu-baseline --no-secondary > /dev/null 2>&1
done
bash tools/ncu_full.sh motion720 motion_m3_kernel
bash tools/ncu_full.sh motion4k motion_m3_kernel
bash tools/ncu_full.sh dpd1 dpd_main_kernel
bash tools/ncu_full.sh dpd3 dpd_main_kernel
bash tools/ncu_full.sh dpd5 dpd_main_kernel
for w in motion720 motion720gray motion4k dpd1 dpd3 dpd5; do
  ncu -i gpurun_out/prof_$w.ncu-rep --page raw --csv > gpurun_out/prof_${w}_raw.csv 2>/dev/null
done
