#!/bin/bash
# compute-sanitizer memcheck, racecheck and synccheck over the whole GPU parity file
# (every case, all four prefix paths: mma.sync, tcgen05, row groups, and the
# shapes each path's tests build).  Output: gpurun_out/san_full/
set -u
cd "$(dirname "$0")/.."
O=gpurun_out/san_full; mkdir -p $O
for tool in ${TOOLS:-memcheck racecheck synccheck}; do
  extra=""
  [ "$tool" = racecheck ] && extra="--racecheck-report analysis"
  timeout 3000 compute-sanitizer --tool $tool $extra --target-processes all --print-limit 200 \
    python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider > $O/$tool.log 2>&1
  echo "$tool rc=$?" >> $O/$tool.log
  grep -E "passed|failed|SUMMARY|rc=" $O/$tool.log | tail -4
done
