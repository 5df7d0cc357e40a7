#!/bin/bash
mkdir -p gpurun_out
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench4.json 2> gpurun_out/bench4.err; echo "bench rc=$?"
SRK_WS_BATCH=8 SRK_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --steps 1 --warmup 3 --no-cpu-baseline \
  > gpurun_out/bench_2ranks.json 2> gpurun_out/bench_2ranks.err; echo "2-rank rc=$?"
