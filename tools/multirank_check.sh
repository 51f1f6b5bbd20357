#!/bin/bash
# Functional check of bench.py's N>1 path (frame-range / block-range shards,
# P2P halo exchange, max-over-ranks timing) on a 1-GPU box: 2 ranks share
# cuda:0 over gloo (NCCL refuses two ranks on one GPU).  Numbers from this
# run are not bench values.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for w in ${MR_WORKLOADS:-motion720 dpd1 dpd3 dpd5}; do
  DF_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --workload $w --steps 3 --warmup 3 \
    > gpurun_out/mr_$w.json 2> gpurun_out/mr_$w.err
  echo "$w rc=$?" >> gpurun_out/mr_status.txt
done
