#!/bin/bash
# Wide merge with one memory round trip: parity, small-fan-out A/B, timelines.
cd "$(dirname "$0")/../../.."
O=gpurun_out/wide; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "merge_many or single_request or tiny or ragged or nested_three" > $O/parity.log 2>&1; echo "rc=$?" >> $O/parity.log
tail -2 $O/parity.log
A=.ab/libforkattn_head.so B=paper_2405_19888_b200/libforkattn.so FANOUTS=1,2,4,8,16 ROUNDS=2 bash profiles/fanout_lib_ab.sh > $O/fanout_ab.log 2>&1
cat $O/fanout_ab.log
bash profiles/build_tl.sh > /dev/null 2>&1 || echo "tl build failed"
for s in 6000,1,256 6000,8,256; do
  echo "== $s isolated"; timeout 300 python profiles/cta_timeline.py --shape $s --isolated 2>&1 | tail -6
done > $O/timeline.log 2>&1
grep -v "^last layer prefix\|^-$" $O/timeline.log
