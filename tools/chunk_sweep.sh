#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/chunk_sweep.txt
for c in 128 32 64 96 192 128; do
  echo "chunk $c" >> gpurun_out/chunk_sweep.txt
  SRK_NTT_CHUNK=$c python tools/ntt_sweep.py >> gpurun_out/chunk_sweep.txt 2>&1
done
cat gpurun_out/chunk_sweep.txt
