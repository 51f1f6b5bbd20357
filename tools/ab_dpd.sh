#!/bin/bash
# A/B of DPD kernel variants (paper_1611_03226_b200/variants/*.so): parity tests per
# variant, then each variant benchmarked twice, interleaved.  -> gpurun_out/ab_dpd.txt
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/ab_dpd.txt
for v in paper_1611_03226_b200/variants/*.so; do
  DF_CUDA_LIB=$PWD/$v timeout 600 python -m pytest tests/test_dpd_gpu.py -q -x 2>&1 | tail -1 | sed "s|^|$(basename $v) tests: |" >> gpurun_out/ab_dpd.txt
done
for rep in 1 2; do
for v in paper_1611_03226_b200/variants/*.so; do
  for w in ${AB_WORKLOADS:-dpd1 dpd3 dpd5}; do
    r=$(DF_CUDA_LIB=$PWD/$v timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-secondary 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['ms_per_step'], d['roofline']['frac'])")
    echo "$(basename $v) $w $r" >> gpurun_out/ab_dpd.txt
  done
done
done
