#!/bin/bash
# Evidence for profiles/<round>/ (run on the GPU box from the repo root):
# full bench line, per-kernel DRAM roofline of one primitive step, the forward
# NTT's DRAM traffic, and --set full summaries (stalls, occupancy) of the top
# kernels.  .ncu-rep files stay in /tmp on the box (gpurun copies back <= 64 MiB).
set -u
out=gpurun_out/prof
rep=/tmp/srk_prof
mkdir -p $out $rep
python bench.py > $out/bench_full.json 2> $out/bench_full.err; echo "bench rc=$?"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --profile-from-start off --csv --log-file $out/launches_step64.csv python tools/prof_prims.py step 64 1 \
    > $out/ncu_step.log 2>&1; echo "ncu step rc=$?"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --profile-from-start off --csv --log-file $out/launches_fwd64.csv python tools/prof_prims.py fwd 64 1 \
    > $out/ncu_fwd.log 2>&1; echo "ncu fwd rc=$?"
ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:ntt_pass_kernel \
    -c 6 -f -o $rep/ntt_fwd_full python tools/prof_prims.py fwd 64 1 > $out/ncu_fwd_full.log 2>&1; echo "ncu full rc=$?"
python tools/ncu_summary.py $rep/ntt_fwd_full.ncu-rep > $out/ncu_full_fwd_ntt.txt
ncu --set full --import-source on --clock-control none --profile-from-start off \
    -k regex:"k_ks_combine|k_moddown_conv|k_modup|k_ks_inner|k_moddown_v" -c 8 -f -o $rep/rot_full \
    python tools/prof_prims.py rot 8 1 > $out/ncu_rot_full.log 2>&1; echo "ncu rot rc=$?"
python tools/ncu_summary.py $rep/rot_full.ncu-rep > $out/ncu_full_rotation.txt
du -sh gpurun_out
