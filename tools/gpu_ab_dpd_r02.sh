# round-2 DPD A/B session: parity of every variant, then interleaved bench lines,
# then the traced variant's timeline.  -> gpurun_out/ab_dpd.txt, gpurun_out/dpd_trace.txt
set -x
mkdir -p gpurun_out
rm -f paper_1611_03226_b200/variants/*T.so.keep
for v in paper_1611_03226_b200/variants/*T.so; do mv $v $v.keep; done
AB_WORKLOADS="${AB_WORKLOADS:-dpd1 dpd3}" bash tools/ab_dpd.sh
for v in paper_1611_03226_b200/variants/*T.so.keep; do mv $v ${v%.keep}; done
cat gpurun_out/ab_dpd.txt
: > gpurun_out/dpd_trace.txt
for v in paper_1611_03226_b200/variants/*T.so; do
  for wl in dpd1 dpd3; do
    echo "== $(basename $v) $wl" >> gpurun_out/dpd_trace.txt
    DF_CUDA_LIB=$PWD/$v python tools/probe_dpd_trace.py $wl 2>&1 | tail -13 >> gpurun_out/dpd_trace.txt
  done
done
cat gpurun_out/dpd_trace.txt
