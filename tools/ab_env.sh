#!/bin/bash
# Generic environment-knob A/B of graphed decode steps (ctx 1024), two rounds:
#   bash tools/ab_env.sh "X=0" "WS_SK_SPLITJ=1" "WS_DEC_CLUSTER=8" ...
for r in 1 2; do
for e in "$@"; do
  echo "[$e]"
  env $e timeout 300 python tools/decode_profile.py --graphed --back-to-back --ctx 1024 --batch ${AB_BATCH:-1,4,16,64} --steps 40 | cut -c1-70
done
done
