#!/bin/bash
# TC_BOUNDARY_COST on the other configs (4 interleaved rounds).
cd "$(dirname "$0")/../../.."
O=gpurun_out/tune3; mkdir -p $O
L=paper_2405_19888_b200/libforkattn.so
for CFG in llama13b_p6000_b256 llama7b_p6000_b64 mapreduce_13b nested_13b llama13b_p6000_b64; do
for opt in TC_BOUNDARY_COST=12 TC_BOUNDARY_COST=16; do
  timeout 400 python profiles/lib_ab.py --a $L --b $L --opt-b $opt --rounds 4 --config $CFG > $O/${CFG}_$opt.log 2>&1
  echo "$CFG $opt $(tail -n 2 $O/${CFG}_$opt.log | tr '\n' ' ')"
done; done | tee $O/summary.txt
