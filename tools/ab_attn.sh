# A/B builds of the prefill attention kernel: each line of $VARIANTS is a set
# of env assignments for the build (e.g. "WS_ATTN_PINGPONG=0 WS_ATTN_POLY=3")
echo "$VARIANTS" | while read -r v; do
  [ -z "$v" ] && continue
  env $v python -m paper_2512_09472_b200.build -f > /dev/null
  echo -n "[$v] "; python tools/attn_bench.py --check --iters 100
done
python -m paper_2512_09472_b200.build -f > /dev/null
