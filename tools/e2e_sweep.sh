#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/e2e_sweep.txt
for c in 6 4 8 10 12; do
  SRK_E2E_CHUNKS=$c python bench.py --steps 5 --warmup 3 --no-pipelines --no-cpu-baseline 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('chunks $c', d['ms_per_step'], d['e2e']['ms_per_step'], d['e2e']['pipeline'])" >> gpurun_out/e2e_sweep.txt
done
cat gpurun_out/e2e_sweep.txt
