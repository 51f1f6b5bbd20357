cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
AB_WORKLOADS="motion720 motion4k motion720gray" bash tools/ab_motion.sh
for v in t2 t3; do
  DF_CUDA_LIB=$PWD/paper_1611_03226_b200/variants/libdf_cuda_$v.so timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:motion_m3 -s 3 -c 1 --csv python bench.py --workload motion720 --steps 1 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/ncu_$v.csv 2>/dev/null
done
