#!/bin/bash
# Short-prompt prefill with the attention kernel chosen by length (default)
# vs the tcgen05 kernels throughout (WS_ATTN_SHORT_MMA=0).
timeout 1200 python -m pytest tests/test_gpu_model.py tests/test_gpu_attention.py -q -m gpu -x 2>&1 | tail -2
for v in "X=0" "WS_ATTN_SHORT_MMA=0"; do
  for m in llama3-8b phi3-mini qwen2.5-7b; do
    for t in 64 128 256 384 512; do
      echo -n "[$v] $m $t: "; env $v timeout 300 python tools/prefill_profile.py --model $m --tokens $t --iters 8 | tail -1
    done
  done
done
