#!/bin/bash
timeout 1200 python -m pytest tests/test_gpu_model.py tests/test_gpu_attention.py -q -m gpu -x 2>&1 | tail -2
for r in 1 2; do python tools/decode_profile.py --graphed --back-to-back --ctx 1024 --batch 1,8,16,32,64 --steps 40 | cut -c1-60; done
for t in 16 64 128; do echo -n "prefill $t: "; python tools/prefill_profile.py --tokens $t --iters 8 | tail -1; done
