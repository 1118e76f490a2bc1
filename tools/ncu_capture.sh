#!/bin/bash
# ncu evidence for profiles/ (one GPU; never a multi-rank command):
#  1. per-launch time + DRAM bytes of one decode step (C2, C3, C4), caches kept
#     warm across launches as in the real chain (--cache-control none);
#  2. --set full captures of one layer's decode kernels of C2 and of the
#     lm_head + argmax GEMM, one C4 beam-attention launch, one tcgen05 prefill
#     attention launch.
# usage: tools/ncu_capture.sh [tag]   (outputs gpurun_out/ncu_step_<w>.csv, *.ncu-rep)
tag=${1:-r2}
mkdir -p gpurun_out
for w in c2 c3 c4; do
  ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --cache-control none --clock-control none --csv --log-file gpurun_out/ncu_step_$w.csv \
      python tools/one_step.py $w > gpurun_out/one_step_$w.log 2>&1
  python tools/step_profile.py gpurun_out/ncu_step_$w.csv > gpurun_out/step_profile_$w.txt 2>&1
done
ncu --nvtx --nvtx-include "step/" --set full --import-source on --clock-control none -c 6 \
    -o gpurun_out/prof_layer_c2_$tag python tools/one_step.py c2 > /dev/null 2>&1
ncu --nvtx --nvtx-include "step/" --set full --import-source on --clock-control none -k regex:gemm_tc_kernel \
    -s 48 -c 1 -o gpurun_out/prof_lm_head_c2_$tag python tools/one_step.py c2 > /dev/null 2>&1
ncu --nvtx --nvtx-include "step/" --set full --import-source on --clock-control none -k regex:attn_decode_beam \
    -c 1 -o gpurun_out/prof_attn_beam_c4_$tag python tools/one_step.py c4 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:attn_prefill_tc -s 3 -c 1 \
    -o gpurun_out/prof_pfattn_tc_$tag python tools/pf_attn_once.py 128 > /dev/null 2>&1
ls -la gpurun_out
