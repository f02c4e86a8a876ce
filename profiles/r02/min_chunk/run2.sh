#!/bin/bash
# Beside a prefix grid: minimum chunk 2 (B) vs 4 (A); parity; headline unchanged.
cd "$(dirname "$0")/../../.."
O=gpurun_out/mc2; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tc" > $O/parity.log 2>&1; echo "rc=$?" >> $O/parity.log
tail -2 $O/parity.log
A=.ab/libforkattn_head.so B=paper_2405_19888_b200/libforkattn.so FANOUTS=2,8,12,16,24,32,48 ROUNDS=2 bash profiles/fanout_lib_ab.sh > $O/fanout_ab.log 2>&1
cat $O/fanout_ab.log
timeout 600 python profiles/lib_ab.py --a .ab/libforkattn_head.so --b paper_2405_19888_b200/libforkattn.so --rounds 2 --config mapreduce_13b > $O/ab_mr.log 2>&1; tail -2 $O/ab_mr.log
