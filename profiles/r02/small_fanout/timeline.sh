#!/bin/bash
# CTA timelines of small fan-outs (debug build profiles/build/libforkattn_tl.so)
cd "$(dirname "$0")/../../.."
O=gpurun_out/sf_tl; mkdir -p $O
for s in 6000,1,256 6000,4,256 6000,8,256 6000,64,256; do
  echo "== $s chained"; timeout 300 python profiles/cta_timeline.py --shape $s 2>&1 | tail -12
  echo "== $s isolated"; timeout 300 python profiles/cta_timeline.py --shape $s --isolated 2>&1 | tail -12
done > $O/timeline.log 2>&1
cat $O/timeline.log
