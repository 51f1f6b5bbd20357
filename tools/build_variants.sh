#!/bin/bash
# Builds libdf_cuda.so variants of one translation unit for GPU A/B runs:
#   tools/build_variants.sh motion "R50_E1:-DDF_MOTION_R=50 -DDF_MOTION_EDGE_SPLIT=1" ...
# Output: paper_1611_03226_b200/variants/libdf_cuda_<name>.so (select with DF_CUDA_LIB).
set -e
cd "$(dirname "$0")/../paper_1611_03226_b200/csrc"
make -s >/dev/null
unit=$1; shift
mkdir -p ../variants build/var
rm -f ../variants/*.so
NVFLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC,-O2 -I../../include --expt-relaxed-constexpr"
others=$(ls build/*.o | grep -v "build/$unit.o")
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  ( nvcc $NVFLAGS $flags -c $unit.cu -o build/var/${unit}_$name.o &&
    nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../variants/libdf_cuda_$name.so $others build/var/${unit}_$name.o -lcudart ) &
done
wait
ls ../variants
