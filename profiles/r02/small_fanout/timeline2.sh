#!/bin/bash
cd "$(dirname "$0")/../../.."
O=gpurun_out/sf_tl; mkdir -p $O
for s in 6000,1,256 6000,8,256; do
  echo "== $s chained"; timeout 300 python profiles/cta_timeline.py --shape $s 2>&1 | tail -6
  echo "== $s isolated"; timeout 300 python profiles/cta_timeline.py --shape $s --isolated 2>&1 | tail -6
done > $O/timeline2.log 2>&1
cat $O/timeline2.log
