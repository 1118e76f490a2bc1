#!/bin/bash
# ncu evidence for profiles/: the launch list of one C2 bench step and --set full
# captures of the top decode kernels (one GPU; never a multi-rank command).
mkdir -p gpurun_out
rm -f gpurun_out/*.ncu-rep gpurun_out/launches.csv
ncu --metrics gpu__time_duration.sum --clock-control none -s 400 -c 100 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
# decode step kernels via the graph-replayed trace tool (skip the prefill launches)
ncu --set full --clock-control none --import-source on -k regex:attn_decode_split -s 20 -c 1 \
    -o gpurun_out/prof_attn_decode_split python tools/trace_step.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 2 -c 1 \
    -o gpurun_out/prof_lm_head python tools/lm_once.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 2 -c 1 \
    -o gpurun_out/prof_prefill_gemm python tools/pf_once.py > /dev/null 2>&1
ls -la gpurun_out
