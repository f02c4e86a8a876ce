#!/bin/bash
# Interleaved A/B of two source trees on one box: ./ (new) against .ab/old
# (a built copy of an earlier commit).  Usage: bash profiles/ab_tree.sh [config] [reps]
cd "$(dirname "$0")/.."
cfg=${1:-llama13b_p6000_b64}; reps=${2:-3}
mkdir -p gpurun_out
for i in $(seq $reps); do
  for t in old new; do
    d=.; [ $t = old ] && d=.ab/old
    (cd $d && python bench.py --config $cfg --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-check --no-isolated 2>/dev/null) \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$t', round(d['value']), round(r['layer_us'],2), round(r['frac'],4), d['clocks']['sm_mhz'])"
  done
done
