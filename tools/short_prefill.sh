#!/bin/bash
for t in 255 256; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pre_l_$t.csv \
    python tools/prefill_profile.py --tokens $t --iters 2 > /dev/null 2>&1
  echo "== $t"; python tools/summarize_launches.py gpurun_out/pre_l_$t.csv | head -6
  echo -n "live: "; python tools/prefill_profile.py --tokens $t --iters 8 | tail -1
done
