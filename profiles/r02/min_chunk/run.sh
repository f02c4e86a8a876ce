#!/bin/bash
# Auto minimum chunk for small plans without a prefix grid: parity, fan-out A/B.
cd "$(dirname "$0")/../../.."
O=gpurun_out/mcauto; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "grp or tc" > $O/parity.log 2>&1; echo "rc=$?" >> $O/parity.log
tail -2 $O/parity.log
A=.ab/libforkattn_head.so B=paper_2405_19888_b200/libforkattn.so FANOUTS=1,2,3,4,5,6,7,8 ROUNDS=2 bash profiles/fanout_lib_ab.sh > $O/fanout_ab.log 2>&1
cat $O/fanout_ab.log
