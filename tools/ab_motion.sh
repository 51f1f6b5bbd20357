#!/bin/bash
# A/B of motion kernel variants (paper_1611_03226_b200/variants/*.so, built by
# tools/build_variants.sh): parity tests per variant, then each variant
# benchmarked twice, interleaved.  -> gpurun_out/ab.txt
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/ab.txt
for v in paper_1611_03226_b200/variants/*.so; do
  DF_CUDA_LIB=$PWD/$v timeout 300 python -m pytest tests/test_motion_gpu.py -q -x 2>&1 | tail -1 | sed "s|^|$(basename $v) tests: |" >> gpurun_out/ab.txt
done
for rep in 1 2; do
for v in paper_1611_03226_b200/variants/*.so; do
  for w in ${AB_WORKLOADS:-motion720 motion4k}; do
    r=$(DF_CUDA_LIB=$PWD/$v timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-secondary 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['ms_per_step'], d['roofline']['frac'])")
    echo "$(basename $v) $w $r" >> gpurun_out/ab.txt
  done
done
done
