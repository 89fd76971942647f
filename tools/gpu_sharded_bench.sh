#!/bin/bash
# The bench's N>1 code path in a world of one (the lease has one GPU): torchrun, NCCL
# process group, dehaze_sharded steps, max-over-ranks reductions, the JSON line.
mkdir -p gpurun_out
for c in c3 c4 c2; do
  DHZ_BENCH_SHARDED=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 \
    --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --config $c --steps 5 --warmup 3 \
    --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_sharded_$c.json 2> gpurun_out/bench_sharded_$c.err
  echo "rc=$?"; tail -c 1500 gpurun_out/bench_sharded_$c.json; tail -3 gpurun_out/bench_sharded_$c.err
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29518 \
  bench.py --impl reference --gpus 1 --steps 1 --warmup 1 | tail -c 600
