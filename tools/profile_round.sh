#!/bin/bash
# ncu evidence for profiles/: launch lists (gpu__time_duration) + one --set full per top kernel,
# and the device-resident network kernel (net_kernel, the reference's DPD network shape).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for w in motion720 motion720gray motion4k dpd1 dpd3 dpd5; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$w.csv \
     python bench.py --workload $w --steps 2 --warmup 3 --no-cpu-baseline --no-secondary > /dev/null 2>&1
done
bash tools/ncu_full.sh motion720 motion_m3_kernel
bash tools/ncu_full.sh motion720gray motion_m3_kernel
bash tools/ncu_full.sh motion4k motion_m3_kernel
bash tools/ncu_full.sh dpd1 dpd_wave_kernel
bash tools/ncu_full.sh dpd3 dpd_main_kernel
bash tools/ncu_full.sh dpd5 dpd_main_kernel
timeout 900 ncu --set full --clock-control none --import-source on -k regex:net_kernel -c 1 -o gpurun_out/prof_resident -f \
  python -c "import bench; print(bench.resident_networks())" > gpurun_out/ncu_resident.log 2>&1
for w in motion720 motion720gray motion4k dpd1 dpd3 dpd5 resident; do
  ncu -i gpurun_out/prof_$w.ncu-rep --page raw --csv > gpurun_out/prof_${w}_raw.csv 2>/dev/null
done
