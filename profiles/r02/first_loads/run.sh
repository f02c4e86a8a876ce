#!/bin/bash
# Private stream: chunk A's first loads before the ticket round trip for chunk B.
cd "$(dirname "$0")/../../.."
O=gpurun_out/first; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tc or grp" > $O/parity.log 2>&1; echo "rc=$?" >> $O/parity.log
tail -2 $O/parity.log
A=.ab/libforkattn_head.so; B=paper_2405_19888_b200/libforkattn.so
timeout 600 python profiles/lib_ab.py --a $A --b $B --rounds 4 > $O/ab_b64.log 2>&1; tail -2 $O/ab_b64.log
timeout 600 python profiles/lib_ab.py --a $A --b $B --rounds 3 --config llama13b_p6000_b128 > $O/ab_b128.log 2>&1; tail -2 $O/ab_b128.log
timeout 600 python profiles/lib_ab.py --a $A --b $B --rounds 3 --config nested_13b > $O/ab_nested.log 2>&1; tail -2 $O/ab_nested.log
A=$A B=$B FANOUTS=1,4,16 ROUNDS=2 bash profiles/fanout_lib_ab.sh > $O/fanout_ab.log 2>&1; cat $O/fanout_ab.log
