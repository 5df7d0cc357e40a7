#!/bin/bash
# launch list of the warm packed N=1024 sort + --set full of its base-conversion kernels
mkdir -p gpurun_out/prof /tmp/rep
python tools/prof_pipe.py psort1024 > gpurun_out/prof/psort_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --profile-from-start off --csv --log-file gpurun_out/prof/launches_psort1024.csv python tools/prof_pipe.py psort1024 \
    > gpurun_out/prof/ncu_psort.log 2>&1
echo "launches rc=$?"
python tools/kernel_roofline.py gpurun_out/prof/launches_psort1024.csv gpurun_out/prof/kernel_roofline_psort1024.json "tools/prof_pipe.py psort1024" > gpurun_out/prof/launches_psort1024.txt
ncu --set full --import-source on --clock-control none --profile-from-start off --kernel-name-base mangled \
    -k regex:"k_modup_conv|k_moddown_conv" -c 4 -f -o /tmp/rep/bconv python tools/prof_pipe.py psort1024 \
    > gpurun_out/prof/ncu_bconv.log 2>&1
echo "bconv rc=$?"
python tools/ncu_summary.py /tmp/rep/bconv.ncu-rep > gpurun_out/prof/ncu_full_bconv.txt
python tools/pipe_util.py /tmp/rep/bconv.ncu-rep gpurun_out/prof/bconv_pipe_util.json "ncu --set full -k k_modup_conv|k_moddown_conv: python tools/prof_pipe.py psort1024" > /dev/null
