# In-situ decode split-K sweep (TF_SPLITS="q,o,f1,f2", 0 = auto): bench value and graph-replayed step.
# usage: tools/split_sweep_c2.sh [workload] "q,o,f1,f2" ...
w=${1:-c2}; shift
for sp in "$@"; do
  TF_SPLITS=$sp timeout 300 python bench.py --workload $w --no-cpu-baseline > gpurun_out/sw.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/sw.log').read().strip().splitlines()[-1]); print('$w $sp', round(d['value']), round(d['decode_step']['us'],1))" || tail -3 gpurun_out/sw.log
done
