#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_primitives.py tests/test_gpu_baseline_configs.py -q -x -k "keyswitch or batched or cfg2 or pointer or cfg1" > gpurun_out/ws_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/ws_tests.log
if grep -q "tests rc=0" gpurun_out/ws_tests.log; then timeout 600 bash tools/sweep2.sh; fi
