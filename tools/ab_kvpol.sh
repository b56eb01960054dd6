#!/bin/bash
# Decode-attention K/V L2 policy A/B builds (WS_DEC_KVPOL 0 / 1 evict_first /
# 2 evict_last), graphed decode steps at ctx 1024, two rounds.
for r in 1 2; do
for v in 0 1 2; do
  WS_DEC_KVPOL=$v python -m paper_2512_09472_b200.build -f > /dev/null 2>&1
  echo "[kvpol $v]"; timeout 300 python tools/decode_profile.py --graphed --back-to-back --ctx 1024 --batch 1,16,64 --steps 40 | cut -c1-70
done
done
python -m paper_2512_09472_b200.build -f > /dev/null 2>&1
