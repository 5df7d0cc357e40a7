#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests/test_gpu_pipelines.py tests/test_gpu_baseline_configs.py -q -x > gpurun_out/ab_tmp_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/ab_tmp_tests.log
python bench.py --steps 3 --warmup 3 --quick --no-cpu-baseline 2>gpurun_out/ab_tmp.err | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); P=d['pipelines']; print([(k, round(v['latency_s']*1e3,2), round(v['graph_replay_s']*1e3,2), v['exact_ranks'], v.get('max_rank_err'), v['cost']['ctct_mults'] if 'cost' in v else None) for k,v in P.items()])"
tail -3 gpurun_out/ab_tmp.err
