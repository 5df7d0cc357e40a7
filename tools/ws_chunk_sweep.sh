#!/bin/bash
# primitive step against the internal batch chunk (SRK_WS_BATCH) and the NTT chunk
# (SRK_NTT_CHUNK): do the two rotation lanes share their digit reads through L2?
mkdir -p gpurun_out; : > gpurun_out/ws_chunk_sweep.txt
for cfg in "32 128" "16 128" "16 64" "16 32" "8 32" "32 64" "32 128"; do
  set -- $cfg
  echo "ws_batch $1 ntt_chunk $2" >> gpurun_out/ws_chunk_sweep.txt
  SRK_WS_BATCH=$1 SRK_NTT_CHUNK=$2 python bench.py --steps 5 --warmup 3 --no-pipelines --no-cpu-baseline 2>/dev/null \
    | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['ms'], d['roofline_keyswitch']['ms'], d['e2e']['ms_per_step'])" >> gpurun_out/ws_chunk_sweep.txt
done
cat gpurun_out/ws_chunk_sweep.txt
