#!/bin/bash
# Round-2 final evidence on one GPU box (output under gpurun_out/final/):
# GPU test suite, DRAM traffic at each config's timed plan (traffic_all.sh ->
# profiles/traffic.json), bench lines for every config + the reference arm,
# one ncu --set full capture of the headline layer, the launch list, an
# NVTX-filtered launch list, the fan-out sweep, the host-step profile.
set -u
cd "$(dirname "$0")/.."
make -s -C paper_2405_19888_b200/csrc >/dev/null && make -s -C oracle
O=gpurun_out/final
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gputest.log 2>&1; echo "rc=$?" >> $O/gputest.log
bash profiles/traffic_all.sh > $O/traffic_summary.txt 2>&1
for c in llama13b_p6000_b64 llama13b_p6000_b128 llama13b_p6000_b256 llama7b_p6000_b64 mapreduce_13b nested_13b; do
  timeout 600 python bench.py --config $c > $O/bench_$c.jsonl 2> $O/bench_$c.err
done
timeout 300 python bench.py --impl reference > $O/bench_reference.jsonl 2>&1
FK_NCU_LAYER=1 timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -o $O/headline_full -f python bench.py --no-cpu-baseline --no-e2e --no-isolated --no-check \
  > $O/headline_full.log 2>&1
ncu -i $O/headline_full.ncu-rep --page raw --csv > $O/headline_full_raw.csv 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
  --no-isolated --no-check > /dev/null 2>&1
timeout 600 ncu --nvtx --nvtx-include "fk_attn_decode_layers/" --metrics gpu__time_duration.sum --clock-control none \
  -c 12 --csv --log-file $O/launches_nvtx.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
  --no-isolated --no-check > /dev/null 2>&1
timeout 900 python profiles/fanout_sweep.py --fanouts 1,2,4,8,16,32,64,128,256 > $O/fanout_sweep.log 2>&1
timeout 300 python profiles/host_step.py > $O/host_mgr8.log 2>&1
timeout 300 python profiles/host_step.py --direct > $O/host_direct.log 2>&1
tail -n 8 $O/traffic_summary.txt; tail -n 2 $O/gputest.log
