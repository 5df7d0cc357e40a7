#!/bin/bash
# source-level ncu capture of the plain forward FP64 NTT passes (64-ct batch)
mkdir -p gpurun_out/prof /tmp/rep
ncu --set full --import-source on --clock-control none --profile-from-start off --kernel-name-base mangled \
    -k regex:"ntt_pass_kernelILi8ELb0ELb(0|1)ELi0ELi1ELi16E" -c 4 -f -o /tmp/rep/fwd_ntt python tools/prof_prims.py fwd 64 1 > gpurun_out/prof/ncu_fwd.log 2>&1
echo "rc=$?"
cp /tmp/rep/fwd_ntt.ncu-rep gpurun_out/prof/
