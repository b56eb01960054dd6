#!/bin/bash
# Mid-length prefills: residual GEMMs k-sliced below one wave (default) vs not (WS_TAIL_SLICES=0).
timeout 1200 python -m pytest tests/test_gpu_model.py -q -m gpu -x 2>&1 | tail -2
for v in "X=0" "WS_TAIL_SLICES=0"; do
  for m in 256 384 512 768 1024 2048; do echo -n "[$v] gemm $m "; env $v python tools/gemm_bench.py --m $m --only o,down; done
  for m in llama3-8b phi3-mini; do
    for t in 192 256 512 1000 2048; do
      echo -n "[$v] $m $t: "; env $v timeout 300 python tools/prefill_profile.py --model $m --tokens $t --iters 8 | tail -1
    done
  done
done
