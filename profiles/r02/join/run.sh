#!/bin/bash
# FK_OPT_PREFIX_JOINS experiment: parity of the join path, then option A/Bs
# on one build (arm A = default, arm B = joins).
set -x
cd "$(dirname "$0")/../../.."
O=gpurun_out/join; mkdir -p $O
L=paper_2405_19888_b200/libforkattn.so
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "join" > $O/parity.log 2>&1; echo "parity rc $?" >> $O/parity.log
tail -3 $O/parity.log
timeout 600 python profiles/lib_ab.py --a $L --b $L --opt-b PREFIX_JOINS=1 > $O/ab_b64.log 2>&1
timeout 600 python profiles/lib_ab.py --a $L --b $L --opt-b PREFIX_JOINS=1 --opt-b LAUNCH_ORDER=1 > $O/ab_b64_o1.log 2>&1
timeout 600 python profiles/lib_ab.py --a $L --b $L --opt-b PREFIX_JOINS=1 --config llama13b_p6000_b128 > $O/ab_b128.log 2>&1
timeout 600 python profiles/lib_ab.py --a $L --b $L --opt-b PREFIX_JOINS=1 --config mapreduce_13b > $O/ab_mr.log 2>&1
timeout 600 python profiles/lib_ab.py --a $L --b $L --opt-b PREFIX_JOINS=1 --config nested_13b > $O/ab_nested.log 2>&1
tail -n 2 $O/ab_*.log
