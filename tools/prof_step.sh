#!/bin/bash
# launch list (time + DRAM bytes per kernel) of one primitive step on 64 ciphertexts
set -u
out=gpurun_out/step; mkdir -p $out
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --profile-from-start off --csv"
python tools/prof_prims.py step 64 1 > /dev/null 2>&1 && \
ncu $M --log-file $out/launches_step64.csv python tools/prof_prims.py step 64 1 > $out/ncu_step.log 2>&1; echo "step rc=$?"
python tools/kernel_roofline.py $out/launches_step64.csv $out/kernel_roofline_step64.json "tools/prof_prims.py step 64 1" "--cache-control none" > $out/launches_step64.txt
