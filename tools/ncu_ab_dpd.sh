cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in old s16; do
  for w in dpd1 dpd3; do
    DF_CUDA_LIB=$PWD/paper_1611_03226_b200/variants/libdf_cuda_$v.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:"dpd_(main|warp)_kernel" -s 3 -c 1 \
      -o gpurun_out/ab_${v}_$w -f python bench.py --workload $w --steps 1 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/ab_ncu_${v}_$w.log 2>&1
    ncu -i gpurun_out/ab_${v}_$w.ncu-rep --page raw --csv > gpurun_out/ab_${v}_${w}_raw.csv 2>/dev/null
  done
done
ls -la gpurun_out
