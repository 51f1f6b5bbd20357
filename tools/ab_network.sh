#!/bin/bash
# A/B of the on-device network step (tools/probe_network.py) and the bare motion firing per libdf_cuda variant.
cd "$(dirname "$0")/.."
for rep in 1 2; do
for v in paper_1611_03226_b200/variants/*.so; do
  echo "== $(basename $v) rep $rep"
  DF_CUDA_LIB=$PWD/$v timeout 300 python tools/probe_network.py 2>&1 | tail -4
done
done
