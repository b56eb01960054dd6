#!/bin/bash
# Decode-attention ring depth A/B builds (WS_DEC_STAGES), graphed decode steps.
for r in 1 2; do
for v in 3 2 4; do
  WS_DEC_STAGES=$v python -m paper_2512_09472_b200.build -f > /dev/null 2>&1
  echo "[stages $v]"; python tools/decode_profile.py --graphed --back-to-back --ctx 1024 --batch 1,16,64 --steps 40 | cut -c1-60
done
done
python -m paper_2512_09472_b200.build -f > /dev/null 2>&1
