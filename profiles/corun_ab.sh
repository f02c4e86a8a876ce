#!/bin/bash
# Co-run split tuning per config: the prefix per-SM rate assumption
# (FK_OPT_PREFIX_RATE_PCT, default 50) and the piece-start cost
# (FK_OPT_TC_BOUNDARY_COST, default 4), interleaved (profiles/ab.py).
for c in ${CONFIGS:-llama7b_p6000_b64 llama13b_p6000_b64 nested_13b}; do
  echo "== $c"
  timeout 300 python profiles/ab.py --config $c --rounds 3 --steps 6 \
    --set PREFIX_RATE_PCT=40 --set PREFIX_RATE_PCT=50 --set PREFIX_RATE_PCT=60 --set PREFIX_RATE_PCT=70 2>&1 | tail -4
done
