#!/bin/bash
# Small plans: minimum chunk 2 vs the auto 4 now that the few-rows merge is one round trip.
cd "$(dirname "$0")/../../.."
O=gpurun_out/tune5; mkdir -p $O
for r in 1 2; do
  for o in "" ${OPTS:-"PRIV_MIN_CHUNK=2" "PRIV_MIN_CHUNK=3"}; do
    echo "== round $r opt=$o"
    timeout 300 python profiles/fanout_sweep.py --fanouts ${FANOUTS:-1,2,4,8} --steps 6 ${o:+--opt $o} 2>&1 | \
      python -c "import sys,json; [print(d['fanout'], round(d['tokens_per_s']), round(d['frac'],3), round(d['frac_isolated'],3)) for d in (json.loads(l) for l in sys.stdin if l.startswith('{'))]"
  done
done | tee $O/summary.txt
