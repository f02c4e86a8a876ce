#!/bin/bash
# Default-option check on the final build: each line is an interleaved A/B
# (A = library defaults, B = one option moved) at the headline config.
cd "$(dirname "$0")/../../.."
O=gpurun_out/tune; mkdir -p $O
L=paper_2405_19888_b200/libforkattn.so
CFG=${CFG:-llama13b_p6000_b64}
for opt in PRIV_MIN_CHUNK=1 PRIV_MIN_CHUNK=3 PREFIX_RATE_PCT=40 PREFIX_RATE_PCT=60 TC_BOUNDARY_COST=2 TC_BOUNDARY_COST=8 PRIV_STATIC_FIRST=0 GROUP_FANOUT=0; do
  timeout 400 python profiles/lib_ab.py --a $L --b $L --opt-b $opt --rounds 2 --config $CFG > $O/${CFG}_$opt.log 2>&1
  echo "$opt $(tail -n 2 $O/${CFG}_$opt.log | tr '\n' ' ')"
done | tee $O/${CFG}_summary.txt
