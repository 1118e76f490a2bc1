#!/bin/bash
# ncu captures for profiles/: launch list of one bench step + full sets of the
# top decode kernels. Run under gpurun (one GPU).
set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 200 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
for k in attn_decode_kernel "gemm_tc_kernel<2" "gemm_tc_kernel<5" layernorm_vec; do
  tag=$(echo "$k" | tr -cd 'a-z0-9_')
  ncu --set full --clock-control none --import-source on -k "regex:$k" -s 30 -c 2 \
      -o gpurun_out/prof_$tag python tools/trace_step.py > gpurun_out/ncu_$tag.log 2>&1
done
ls -la gpurun_out
