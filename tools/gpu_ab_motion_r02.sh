# round-2 motion A/B session: parity + interleaved bench lines + per-variant ncu DRAM bytes of the
# top kernel on each workload.  -> gpurun_out/ab.txt, gpurun_out/ab_dram.txt
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
AB_WORKLOADS="${AB_WORKLOADS:-motion720 motion720gray motion4k}" bash tools/ab_motion.sh
: > gpurun_out/ab_dram.txt
for v in paper_1611_03226_b200/variants/*.so; do
  for w in ${AB_WORKLOADS:-motion720 motion720gray motion4k}; do
    DF_CUDA_LIB=$PWD/$v timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
      -k regex:motion_m3_kernel -s 3 -c 1 --csv python bench.py --workload $w --steps 1 --warmup 3 --no-cpu-baseline --no-secondary 2>/dev/null \
      | grep -E "dram__bytes|gpu__time" | awk -F'","' -v v=$(basename $v) -v w=$w '{print v, w, $(NF-2), $(NF-1), $NF}' >> gpurun_out/ab_dram.txt
  done
done
cat gpurun_out/ab.txt gpurun_out/ab_dram.txt
