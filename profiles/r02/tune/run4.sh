#!/bin/bash
# Launch order 1 (private grid first) vs 0 on the headline and x128.
cd "$(dirname "$0")/../../.."
O=gpurun_out/tune4; mkdir -p $O
L=paper_2405_19888_b200/libforkattn.so
for CFG in llama13b_p6000_b64 llama13b_p6000_b128 nested_13b; do
  timeout 400 python profiles/lib_ab.py --a $L --b $L --opt-b LAUNCH_ORDER=1 --rounds 3 --config $CFG > $O/${CFG}_order1.log 2>&1
  echo "$CFG order1 $(tail -n 2 $O/${CFG}_order1.log | tr '\n' ' ')"
done | tee $O/summary.txt
