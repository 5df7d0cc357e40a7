#!/bin/bash
# time tools/ntt_sweep.py for the default library and every variants/lib_*.so
mkdir -p gpurun_out
python tools/ntt_sweep.py > gpurun_out/sweep.txt 2>&1
for l in variants/lib_*.so; do SRK_LIB=$PWD/$l python tools/ntt_sweep.py >> gpurun_out/sweep.txt 2>&1; done
cat gpurun_out/sweep.txt
