#!/bin/bash
# L2 prefetch hint A/B (WS_L2PF bit mask, see ws_model_decode): graphed decode
# steps, ctx 1024, same process layout for every setting, two rounds.
for r in 1 2; do
for cfg in "0" "1" "2" "1 AT1" "5" "13" "29" "4" "8" "16" "29 AT1"; do
  set -- $cfg
  at=0; [ "$2" = "AT1" ] && at=1
  echo "[WS_L2PF=$1 at=$at]"
  WS_L2PF=$1 WS_L2PF_AT=$at timeout 300 python tools/decode_profile.py --graphed --back-to-back --ctx 1024 --batch 1,4,16 --steps 40 | cut -c1-70
done
done
