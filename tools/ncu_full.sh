#!/bin/bash
# ncu --set full of the top kernels (one GPU, short commands)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
W=${1:-motion720}
K=${2:-motion_fused_kernel}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 \
  -o gpurun_out/prof_$W -f python bench.py --workload $W --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_$W.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_$W.log
