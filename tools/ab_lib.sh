#!/bin/bash
# A/B of the shipped library against variants/*.so (SRK_LIB) on the primitive step and the quick pipelines
mkdir -p gpurun_out; : > gpurun_out/ab_lib.txt
python -m pytest tests/test_gpu_primitives.py tests/test_gpu_baseline_configs.py tests/test_gpu_pipelines.py -q -x > gpurun_out/ab_lib_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/ab_lib.txt; tail -2 gpurun_out/ab_lib_tests.log >> gpurun_out/ab_lib.txt
for lib in "" $1 "" $1; do
  echo "lib ${lib:-shipped}" >> gpurun_out/ab_lib.txt
  SRK_LIB=${lib:+$PWD/$lib} python bench.py --steps 10 --warmup 3 --quick --no-cpu-baseline 2>/dev/null \
    | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); P=d['pipelines']; print(d['ms_per_step'], d['roofline']['ms'], d['roofline_inverse_ntt']['ms'], d['roofline_keyswitch']['ms'], d['e2e']['ms_per_step'], [(k, round(v['graph_replay_s']*1e3,2)) for k,v in P.items()])" >> gpurun_out/ab_lib.txt
done
cat gpurun_out/ab_lib.txt
