#!/bin/bash
# compute-sanitizer over the round-2 kernels (one gpurun call) -> gpurun_out/san_r02.txt:
# dpd_wave_kernel (PDL, pre-wait L2 prefetch), the 20-warp M3 motion kernel with alternating chunks,
# the word-wise resident gauss / median actors.
cd "$(dirname "$0")/.."
o=gpurun_out/san_r02.txt; : > $o
run() { echo "## $1" >> $o; shift; timeout 900 "$@" > gpurun_out/san_tmp.log 2>&1; echo "rc=$?" >> gpurun_out/san_tmp.log; grep -E "passed|failed|ERROR SUMMARY|RACECHECK SUMMARY|rc=" gpurun_out/san_tmp.log | tail -4 >> $o; }
run memcheck_dpd compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_dpd_gpu.py -q -x
run racecheck_dpd compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_dpd_gpu.py -q -x -k "chunked or zero_and_impulse or raw_fire or halo"
run synccheck_dpd compute-sanitizer --tool synccheck --error-exitcode 9 python -m pytest tests/test_dpd_gpu.py -q -x -k "chunked or zero_and_impulse or halo"
run memcheck_motion compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_motion_gpu.py -q -x
run racecheck_motion compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_motion_gpu.py -q -x -k "acceptance or fixture or rgb"
run memcheck_resident compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_netrt_gpu.py -q -x -k "motion"
cat $o
