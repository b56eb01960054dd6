#!/bin/bash
# Decode attention split-cluster limit A/B (WS_DEC_CLUSTER), graphed decode steps.
for r in 1 2; do
for v in default 8 4; do
  echo "[cluster $v]"
  if [ $v = default ]; then
    timeout 300 python tools/decode_profile.py --graphed --back-to-back --ctx 1024 --batch 1,4,16 --steps 40 | cut -c1-70
  else
    WS_DEC_CLUSTER=$v timeout 300 python tools/decode_profile.py --graphed --back-to-back --ctx 1024 --batch 1,4,16 --steps 40 | cut -c1-70
  fi
done
done
