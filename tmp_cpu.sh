mkdir -p gpurun_out
python tools/probe_resident.py > gpurun_out/resident.txt 2>&1
for n in 3 5 8; do DF_CPU_NETS=$n python -c "
import bench, json
print($n, json.dumps(bench.cpu_motion(bench.WORKLOADS['motion720'][1], 2, 1)))" >> gpurun_out/cpu_nets.txt 2>&1; done
python -c "
import bench, json
print(json.dumps(bench.cpu_dpd(bench.WORKLOADS['dpd1'][1], 5, 1)))" >> gpurun_out/cpu_nets.txt 2>&1
