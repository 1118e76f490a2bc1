#!/bin/bash
# A/B on one box: bench.py lines for each "NAME=ENV..." spec (no CPU baseline)
# usage: tools/ab.sh <workload> <steps> "base:" "st0:TF_PUSH_ST=0" ...
w=$1; k=$2; shift 2
mkdir -p gpurun_out
for spec in "$@"; do
  name=${spec%%:*}; envs=${spec#*:}
  env $envs python bench.py --workload $w --steps $k --warmup 3 --no-cpu-baseline > gpurun_out/ab_${w}_${name}.json 2> gpurun_out/ab_${w}_${name}.err
  python - "$w" "$name" <<'PY'
import json, sys
w, n = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open(f"gpurun_out/ab_{w}_{n}.json").read().strip().splitlines()[-1])
    pf = d.get("prefill") or {}
    print(f"{w} {n:10s} value {d['value']:9.1f} e2e {d['e2e']['value']:9.1f} step {d['decode_step']['us']:7.1f} us "
          f"prefill {pf.get('us', 0):7.1f} us")
except Exception as e:
    print(w, n, "FAILED", e)
PY
done
