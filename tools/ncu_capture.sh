#!/bin/bash
# ncu evidence for profiles/ (one GPU; never a multi-rank command):
#  1. per-launch time + DRAM bytes of one decode step (C2, C3, C4), caches kept
#     warm across launches as in the real chain (--cache-control none);
#  2. --set full captures of one layer's decode kernels (embed .. FFN2 + LN) and
#     of the lm_head + argmax GEMM of the same step.
set -e
mkdir -p gpurun_out
rm -f gpurun_out/*.ncu-rep gpurun_out/ncu_step_*.csv
for w in c2 c3 c4; do
  ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --cache-control none --clock-control none --csv --log-file gpurun_out/ncu_step_$w.csv \
      python tools/one_step.py $w > gpurun_out/one_step_$w.log 2>&1
  python tools/step_profile.py gpurun_out/ncu_step_$w.csv
done
ncu --nvtx --nvtx-include "step/" --set full --import-source on --clock-control none -c 8 \
    -o gpurun_out/prof_layer_c2 python tools/one_step.py c2 > /dev/null 2>&1
ncu --nvtx --nvtx-include "step/" --set full --import-source on --clock-control none -k regex:gemm_tc_kernel \
    -s 48 -c 1 -o gpurun_out/prof_lm_head_c2 python tools/one_step.py c2 > /dev/null 2>&1
ls -la gpurun_out
