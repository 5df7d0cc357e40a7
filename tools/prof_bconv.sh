#!/bin/bash
# --set full of the base-conversion kernels in the warm packed N=1024 sort
mkdir -p gpurun_out/prof /tmp/rep
for v in ${BCONV_VARIANTS:-1}; do
  SRK_BCONV=$v ncu --set full --import-source on --clock-control none --profile-from-start off \
      -k regex:"k_modup|k_moddown_conv" -c 8 -f -o /tmp/rep/bconv$v python tools/prof_pipe.py psort1024 \
      > gpurun_out/prof/ncu_bconv$v.log 2>&1
  echo "bconv=$v rc=$?"
  python tools/ncu_summary.py /tmp/rep/bconv$v.ncu-rep > gpurun_out/prof/ncu_full_bconv$v.txt
  python tools/pipe_util.py /tmp/rep/bconv$v.ncu-rep gpurun_out/prof/bconv_pipe_util$v.json "bconv=$v" > /dev/null
done
