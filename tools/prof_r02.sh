set -u
out=gpurun_out/prof
mkdir -p $out /tmp/rep
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --profile-from-start off --csv --log-file $out/launches_step64.csv python tools/prof_prims.py step 64 1 > $out/ncu_step.log 2>&1; echo "step rc=$?"
python tools/kernel_roofline.py $out/launches_step64.csv $out/kernel_roofline_step64.json "tools/prof_prims.py step 64 1" > $out/launches_step64.txt
ncu --set full --import-source on --clock-control none --profile-from-start off --kernel-name-base mangled \
    -k regex:"ntt_pass_kernelILi8ELb0ELb0ELi1ELi1ELi16E" -c 6 -f -o /tmp/rep/rot_ntt python tools/prof_prims.py rot 32 1 > $out/ncu_rot.log 2>&1; echo "full rc=$?"
python tools/ncu_summary.py /tmp/rep/rot_ntt.ncu-rep > $out/ncu_full_rot_ntt.txt
cp /tmp/rep/rot_ntt.ncu-rep $out/
