#!/bin/bash
# Narrow merge: the partial count of each warp's second item read before the PDL wait too.
cd "$(dirname "$0")/../../.."
O=gpurun_out/mpf; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "fanout_256 or fullsize or large_fanout or tiny" > $O/parity.log 2>&1; echo "rc=$?" >> $O/parity.log
tail -2 $O/parity.log
A=.ab/libforkattn_head.so; B=paper_2405_19888_b200/libforkattn.so
for c in llama13b_p6000_b128 llama13b_p6000_b256 llama13b_p6000_b64; do
  timeout 600 python profiles/lib_ab.py --a $A --b $B --rounds 4 --config $c > $O/ab_$c.log 2>&1; echo "$c $(tail -n 2 $O/ab_$c.log | tr '\n' ' ')"
done
