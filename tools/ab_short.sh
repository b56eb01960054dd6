#!/bin/bash
# RoPE/KV append in the skinny QKV GEMM's cluster reduce up to 8 (default) / 16 / 32 rows.
for r in 1 2; do
for v in "X=0" "WS_FUSE_ROPE_ROWS=16" "WS_FUSE_ROPE_ROWS=32"; do
  echo "[$v]"; env $v timeout 600 python tools/decode_profile.py --graphed --back-to-back --ctx 1024 --batch 9,16,24,32 --steps 40 | cut -c1-60
  for t in 16 32; do echo -n "  prefill $t: "; env $v timeout 300 python tools/prefill_profile.py --tokens $t --iters 8 | tail -1; done
done
done
