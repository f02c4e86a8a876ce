#!/bin/bash
# compute-sanitizer racecheck + synccheck (+ memcheck) over the GPU parity
# cases on the three prefix paths (mma.sync, tcgen05, row groups in the private kernel) and both merge kernels, final kernels.
# Usage (GPU box): bash profiles/sanitize.sh  -> gpurun_out/sanitize_*.log
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/${SAN_OUT:-.}
SEL='tiny or ragged or nested_three or merge_by_either or stream_k or many_splits or fill_while or merge_many or chunk_queue or two_generations or single_request or attend_own_token_synthetic'
for tool in racecheck synccheck memcheck; do
  extra=""
  [ "$tool" = racecheck ] && extra="--racecheck-report analysis"
  timeout 2400 compute-sanitizer --tool $tool $extra --target-processes all --print-limit 200 \
    python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "$SEL" -p no:cacheprovider \
    > gpurun_out/${SAN_OUT:-.}/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/${SAN_OUT:-.}/sanitize_$tool.log
  tail -4 gpurun_out/${SAN_OUT:-.}/sanitize_$tool.log
done
# the synccheck semantics behind round 1's mma_commit report (profiles/synccheck_repro.cu)
nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/fk_sc_repro profiles/synccheck_repro.cu
for w in 0 1; do
  compute-sanitizer --tool synccheck /tmp/fk_sc_repro $w > gpurun_out/${SAN_OUT:-.}/sanitize_repro_$w.log 2>&1
  echo "repro wait_every=$w rc=$?" >> gpurun_out/${SAN_OUT:-.}/sanitize_repro_$w.log
  grep -E "Missing wait|ERROR SUMMARY|wait_every" gpurun_out/${SAN_OUT:-.}/sanitize_repro_$w.log
done
