#!/bin/bash
# Skinny-GEMM plan check: model parity tests, per-GEMM timings (Llama-3-8B and
# Phi-3 shapes), short prefills of the configs-3/5 request shapes, graphed decode.
timeout 900 python -m pytest tests/test_gpu_model.py -q -m gpu -x 2>&1 | tail -2
timeout 300 python tools/skinny_bench.py --phi 1,16,32,64,128
timeout 300 python tools/skinny_bench.py 1,16,32,64,128
for m in llama3-8b qwen2.5-7b mistral-7b phi3-mini; do
  for t in 16 64 128; do
    echo -n "  $m $t: "; timeout 300 python tools/prefill_profile.py --model $m --tokens $t --iters 10 | tail -1
  done
done
timeout 600 python tools/decode_profile.py --graphed --back-to-back --ctx 1024 --batch 1,16,32,64 --steps 40 | cut -c1-60
