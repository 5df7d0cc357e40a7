#!/bin/bash
# A/B of engine.parallel (the rank's two replications on two streams): SRK_BRANCH=0 runs them in turn
mkdir -p gpurun_out; : > gpurun_out/ab_branch.txt
python -m pytest tests/test_gpu_pipelines.py tests/test_gpu_baseline_configs.py -q -x > gpurun_out/ab_branch_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/ab_branch.txt; tail -2 gpurun_out/ab_branch_tests.log >> gpurun_out/ab_branch.txt
for f in 0 1 0 1; do
  echo "branch $f" >> gpurun_out/ab_branch.txt
  SRK_BRANCH=$f python bench.py --steps 3 --warmup 3 --quick --no-cpu-baseline 2>>gpurun_out/ab_branch.err \
    | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); P=d['pipelines']; print([(k, round(v['latency_s']*1e3,2), round(v['graph_replay_s']*1e3,2), v['exact_ranks']) for k,v in P.items()])" >> gpurun_out/ab_branch.txt
done
cat gpurun_out/ab_branch.txt; tail -5 gpurun_out/ab_branch.err
