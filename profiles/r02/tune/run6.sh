#!/bin/bash
# 7B and nested: prefix rate and boundary cost around the defaults (3 rounds).
cd "$(dirname "$0")/../../.."
O=gpurun_out/tune6; mkdir -p $O
L=paper_2405_19888_b200/libforkattn.so
for CFG in llama7b_p6000_b64 nested_13b; do
for opt in PREFIX_RATE_PCT=45 PREFIX_RATE_PCT=55 TC_BOUNDARY_COST=20; do
  timeout 400 python profiles/lib_ab.py --a $L --b $L --opt-b $opt --rounds 3 --config $CFG > $O/${CFG}_$opt.log 2>&1
  echo "$CFG $opt $(tail -n 2 $O/${CFG}_$opt.log | tr '\n' ' ')"
done; done | tee $O/summary.txt
