#!/bin/bash
# A/B the megakernel tuning knobs on C2 (step time via the trace tool's end stamp)
for cfg in "0 64" "1 64" "1 256" "3 64" "3 512" "2 256"; do
  set -- $cfg
  echo "FLAGS=$1 SLEEP=$2: $(TF_MK_FLAGS=$1 TF_MK_SLEEP=$2 CFG=c2 timeout 200 python tools/mk_check.py 2>&1 | grep 'MEGAKERNEL=1')"
done
