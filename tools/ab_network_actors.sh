#!/bin/bash
# A/B of libdf_cuda.so variants (tools/build_variants.sh netrt ...) on the
# resident motion network (tools/probe_resident_rate.py), after the resident
# network GPU tests on the default build.  VARIANTS="old mb4 ...", DPD=1 adds
# tools/probe_resident_dpd.py.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
P=paper_1611_03226_b200
cp $P/libdf_cuda.so /tmp/default_libdf_cuda.so
timeout 600 python -m pytest tests/test_netrt_gpu.py -q -x > gpurun_out/netrt_tests.log 2>&1; echo "rc=$?" >> gpurun_out/netrt_tests.log
for v in ${VARIANTS:-old mb4 mb8 mb16}; do
  cp $P/variants/libdf_cuda_$v.so $P/libdf_cuda.so
  echo "== $v" >> gpurun_out/ab_net.log
  RATES=${RATES:-1,5,10,30} timeout 300 python tools/probe_resident_rate.py >> gpurun_out/ab_net.log 2>&1
  if [ -n "$DPD" ]; then BRANCH_CTAS=${BRANCH_CTAS:-8,32} timeout 300 python tools/probe_resident_dpd.py >> gpurun_out/ab_net.log 2>&1; fi
done
cp /tmp/default_libdf_cuda.so $P/libdf_cuda.so
