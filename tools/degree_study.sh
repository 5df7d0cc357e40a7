#!/bin/bash
# the degree / comparison-depth study on the GPU (paper_2412_15126_b200/sweep.py)
mkdir -p gpurun_out
python -m paper_2412_15126_b200.sweep --task rank --count 128 --degrees 64 128 256 512 1024 2048 --seeds 3 \
    --json gpurun_out/degree_study_rank128_cheb.json > gpurun_out/degree_study.txt 2>&1
python -m paper_2412_15126_b200.sweep --task rank --count 128 --composite 1,1 2,1 2,2 3,2 4,2 5,2 --seeds 3 \
    --json gpurun_out/degree_study_rank128_composite.json >> gpurun_out/degree_study.txt 2>&1
python -m paper_2412_15126_b200.sweep --task max --count 128 --composite 3,2 4,2 --seeds 2 \
    --json gpurun_out/degree_study_max128_composite.json >> gpurun_out/degree_study.txt 2>&1
cat gpurun_out/degree_study.txt
