#!/bin/bash
# compute-sanitizer over small GPU cases (one tool per gpurun call: TOOL=memcheck|racecheck|synccheck)
TOOL=${TOOL:-memcheck}
mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool $TOOL --error-exitcode 99 --print-limit 20 \
    python -m pytest tests/test_gpu_primitives.py -q -x -k "toy and not chunking" -p no:cacheprovider \
    > gpurun_out/sanitize_${TOOL}.log 2>&1
echo "primitives rc=$?" | tee -a gpurun_out/sanitize_${TOOL}.log
timeout 900 compute-sanitizer --tool $TOOL --error-exitcode 99 --print-limit 20 \
    python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitize_${TOOL}_smoke.log 2>&1
echo "smoke rc=$?" | tee -a gpurun_out/sanitize_${TOOL}_smoke.log
