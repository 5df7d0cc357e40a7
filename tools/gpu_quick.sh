#!/bin/bash
# quick GPU iteration: key-switch parity subset, primitive-step bench, optional profile
set -u
mkdir -p gpurun_out
python -m pytest tests/test_gpu_primitives.py tests/test_gpu_baseline_configs.py -q -x -k "keyswitch or batched or cfg2 or switches or rescale or ntt" > gpurun_out/quick_tests.log 2>&1
echo "tests rc=$?" | tee -a gpurun_out/quick_tests.log
python bench.py --steps 5 --warmup 3 --no-pipelines --no-cpu-baseline > gpurun_out/quick_bench.json 2> gpurun_out/quick_bench.err
echo "bench rc=$?"
if [ "${PROF:-0}" = "1" ]; then bash tools/prof_r02.sh; fi
