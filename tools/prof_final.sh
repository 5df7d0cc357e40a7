#!/bin/bash
# round evidence for profiles/r02 (run on the GPU box from the repo root)
set -u
out=gpurun_out/final; rep=/tmp/rep
mkdir -p $out $rep
python bench.py --steps 20 --warmup 5 > $out/bench_full.json 2> $out/bench_full.err; echo "bench rc=$?"
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --profile-from-start off --csv"
python tools/prof_prims.py step 64 1 > /dev/null 2>&1 && \
ncu $M --log-file $out/launches_step64.csv python tools/prof_prims.py step 64 1 > $out/ncu_step.log 2>&1; echo "step rc=$?"
python tools/kernel_roofline.py $out/launches_step64.csv $out/kernel_roofline_step64.json "tools/prof_prims.py step 64 1" "--cache-control none" > $out/launches_step64.txt
ncu $M --log-file $out/launches_fwd64.csv python tools/prof_prims.py fwd 64 1 > $out/ncu_fwd.log 2>&1; echo "fwd rc=$?"
python tools/kernel_roofline.py $out/launches_fwd64.csv $out/ntt_fwd_traffic.json "tools/prof_prims.py fwd 64 1" "--cache-control none" > $out/launches_fwd64.txt
ncu $M --log-file $out/launches_relin64.csv python tools/prof_prims.py keyswitch 64 1 > $out/ncu_relin.log 2>&1; echo "relin rc=$?"
python tools/kernel_roofline.py $out/launches_relin64.csv $out/relin64_traffic.json "tools/prof_prims.py keyswitch 64 1" "--cache-control none" > $out/launches_relin64.txt
ncu $M --log-file $out/launches_rank128.csv python tools/prof_pipe.py rank > $out/ncu_rank.log 2>&1; echo "rank rc=$?"
python tools/kernel_roofline.py $out/launches_rank128.csv $out/kernel_roofline_rank128.json "tools/prof_pipe.py rank" "--cache-control none" > $out/launches_rank128.txt
ncu --set full --import-source on --clock-control none --profile-from-start off --kernel-name-base mangled \
    -k regex:"ntt_pass_kernelILi8ELb0ELb(0|1)ELi(0|1)ELi1ELi16E" -c 6 -f -o $rep/ntt_full python tools/prof_prims.py rot 32 1 > $out/ncu_full.log 2>&1; echo "full rc=$?"
python tools/ncu_summary.py $rep/ntt_full.ncu-rep > $out/ncu_full_ntt_passes.txt
python tools/pipe_util.py $rep/ntt_full.ncu-rep $out/ntt_pipe_util.json "ncu --set full: FP64 NTT passes (plain column, plain row, key-switch row) of 15 hoisted rotations of 32 ct" > /dev/null
du -sh $out
