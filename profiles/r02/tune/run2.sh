#!/bin/bash
# Second pass on the options the first pass moved (4 interleaved rounds).
cd "$(dirname "$0")/../../.."
O=gpurun_out/tune2; mkdir -p $O
L=paper_2405_19888_b200/libforkattn.so
for CFG in llama13b_p6000_b64 llama13b_p6000_b128; do
for opt in PREFIX_RATE_PCT=60 PREFIX_RATE_PCT=70 TC_BOUNDARY_COST=8 TC_BOUNDARY_COST=12; do
  timeout 400 python profiles/lib_ab.py --a $L --b $L --opt-b $opt --rounds 4 --config $CFG > $O/${CFG}_$opt.log 2>&1
  echo "$CFG $opt $(tail -n 2 $O/${CFG}_$opt.log | tr '\n' ' ')"
done; done | tee $O/summary.txt
