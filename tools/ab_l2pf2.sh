#!/bin/bash
# L2 prefetch hints x evict_first weight streams (WS_L2PF, WS_L2PF_AT, WS_SK_EVF):
# graphed decode steps, ctx 1024, two rounds.
cfgs=${*:-"0:0:0 0:0:1 8:0:1 8:1:1 24:0:1 29:0:1 29:1:1"}
for r in 1 2; do
for cfg in $cfgs; do
  IFS=: read m at evf <<< "$cfg"
  echo "[WS_L2PF=$m at=$at evf=$evf]"
  WS_L2PF=$m WS_L2PF_AT=$at WS_SK_EVF=$evf timeout 300 python tools/decode_profile.py --graphed --back-to-back --ctx 1024 --batch 1,4,16 --steps 40 | cut -c1-70
done
done
