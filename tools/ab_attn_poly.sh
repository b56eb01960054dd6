for P in ${POLYS:-0 1 2}; do
  WS_ATTN_POLY=$P python -m paper_2512_09472_b200.build -f > /dev/null
  echo -n "poly $P/8: "; python tools/attn_bench.py --check --iters 100
done
