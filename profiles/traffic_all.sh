#!/bin/bash
# DRAM traffic of one layer's kernels at the plan bench.py's roofline is timed
# on, for every benchmarked config (ncu, cache control "all": cold L2 per
# kernel, kernels serialised), then profiles/make_traffic_all.py writes
# profiles/traffic.json (read by bench.py: roofline.traffic).
# Usage (GPU box): bash profiles/traffic_all.sh [configs...]
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/traffic
CONFIGS=${@:-llama13b_p6000_b64 llama13b_p6000_b128 llama13b_p6000_b256 llama7b_p6000_b64 mapreduce_13b nested_13b}
for c in $CONFIGS; do
  FK_NCU_LAYER=1 timeout 900 ncu --profile-from-start off --clock-control none \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum \
    --csv --log-file gpurun_out/traffic/$c.csv \
    python bench.py --config $c --no-cpu-baseline --no-e2e --no-isolated --no-check > gpurun_out/traffic/$c.log 2>&1
  cp gpurun_out/ncu_layer.json gpurun_out/traffic/$c.json
  echo "$c rc=$?"
done
python profiles/make_traffic_all.py gpurun_out/traffic
