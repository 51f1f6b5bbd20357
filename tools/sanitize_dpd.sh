#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over the DPD GPU tests (one gpurun call) -> gpurun_out/san_dpd_final.txt
cd "$(dirname "$0")/.."
o=gpurun_out/san_dpd_final.txt; : > $o
run() { echo "## $1" >> $o; shift; timeout 600 "$@" > gpurun_out/san_tmp.log 2>&1; echo "rc=$?" >> gpurun_out/san_tmp.log; grep -E "passed|failed|ERROR SUMMARY|RACECHECK SUMMARY|rc=" gpurun_out/san_tmp.log | tail -4 >> $o; }
run memcheck_dpd compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_dpd_gpu.py -q -x -k "chunked or shard or halo or channel_bound or raw_fire or zero_and_impulse or gating"
run racecheck_dpd compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_dpd_gpu.py -q -x -k "chunked or zero_and_impulse or raw_fire"
run synccheck_dpd compute-sanitizer --tool synccheck --error-exitcode 9 python -m pytest tests/test_dpd_gpu.py -q -x -k "chunked or zero_and_impulse or halo"
