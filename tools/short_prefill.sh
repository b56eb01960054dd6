#!/bin/bash
# Launch lists of short-prompt prefills under two skinny plans.
for v in "X=0" "WS_SKINNY_CLUSTER_MP=64"; do
  for spec in "phi3-mini 64" "llama3-8b 64"; do
    set -- $spec
    env $v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pre_$1_$2_${v%%=*}.csv \
      python tools/prefill_profile.py --model $1 --tokens $2 --iters 2 > /dev/null 2>&1
  done
done
