#!/bin/bash
# e2e step time against the size of the first / last chunk (SRK_E2E_RAMP: first chunk = per / ramp)
mkdir -p gpurun_out; : > gpurun_out/e2e_ramp.txt
for cfg in "6 2" "6 3" "6 4" "6 6" "8 2" "8 4" "5 3" "6 2"; do
  set -- $cfg
  SRK_E2E_CHUNKS=$1 SRK_E2E_RAMP=$2 python bench.py --steps 5 --warmup 3 --no-pipelines --no-cpu-baseline 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('chunks $1 ramp $2', d['ms_per_step'], d['e2e']['ms_per_step'], d['e2e']['pipeline'])" >> gpurun_out/e2e_ramp.txt
done
cat gpurun_out/e2e_ramp.txt
