#!/bin/bash
# A/B: default library vs variants/lib_*.so, two rounds each (ntt_sweep + packed sort)
mkdir -p gpurun_out; : > gpurun_out/sweep2.txt
for r in 1 2; do
  python tools/ntt_sweep.py >> gpurun_out/sweep2.txt 2>&1
  python tools/prof_pipe.py psort1024 >> gpurun_out/sweep2.txt 2>&1
  for l in variants/lib_*.so; do
    SRK_LIB=$PWD/$l python tools/ntt_sweep.py >> gpurun_out/sweep2.txt 2>&1
    SRK_LIB=$PWD/$l python tools/prof_pipe.py psort1024 >> gpurun_out/sweep2.txt 2>&1
  done
done
cat gpurun_out/sweep2.txt
