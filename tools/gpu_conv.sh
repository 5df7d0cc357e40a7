#!/bin/bash
# conversion-kernel iteration: parity subset + primitive sweep + packed sort latency
mkdir -p gpurun_out
python -m pytest tests/test_gpu_primitives.py tests/test_gpu_baseline_configs.py -q -x \
  -k "keyswitch or batched or cfg2 or switches or cfg1 or cfg5_multi_sort_n1024_packed or cfg4" > gpurun_out/conv_tests.log 2>&1
echo "tests rc=$?" | tee -a gpurun_out/conv_tests.log
python tools/ntt_sweep.py > gpurun_out/conv_sweep.txt 2>&1
python tools/prof_pipe.py psort1024 >> gpurun_out/conv_sweep.txt 2>&1
python tools/prof_pipe.py sort1024 >> gpurun_out/conv_sweep.txt 2>&1
cat gpurun_out/conv_sweep.txt
