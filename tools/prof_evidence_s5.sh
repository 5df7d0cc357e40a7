#!/bin/bash
# end-of-round evidence refresh (kernels unchanged since the ncu captures in profiles/r02):
# full bench line, reference arm, full GPU test log
mkdir -p gpurun_out/ev
python bench.py --steps 20 --warmup 5 > gpurun_out/ev/bench_full.json 2> gpurun_out/ev/bench_full.err; echo "bench rc=$?"
python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/ev/bench_reference_arm.json 2> gpurun_out/ev/bench_reference_arm.err; echo "ref rc=$?"
python -m pytest tests -m gpu -q -rA > gpurun_out/ev/gputest_full.log 2>&1; echo "gputest rc=$?"; tail -2 gpurun_out/ev/gputest_full.log
