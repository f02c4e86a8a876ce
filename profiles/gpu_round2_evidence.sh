#!/bin/bash
# Round-2 evidence on one GPU box: bench lines for every config, traffic at
# each timed plan (traffic_all.sh), one ncu --set full capture of the
# headline layer, the launch list.  Output under gpurun_out/r02/.
set -u
cd "$(dirname "$0")/.."
make -s -C paper_2405_19888_b200/csrc >/dev/null && make -s -C oracle
mkdir -p gpurun_out/r02
bash profiles/traffic_all.sh > gpurun_out/r02/traffic_summary.txt 2>&1
for c in llama13b_p6000_b64 llama13b_p6000_b128 llama13b_p6000_b256 llama7b_p6000_b64 mapreduce_13b nested_13b; do
  timeout 600 python bench.py --config $c > gpurun_out/r02/bench_$c.jsonl 2> gpurun_out/r02/bench_$c.err
done
timeout 300 python bench.py --impl reference > gpurun_out/r02/bench_reference.jsonl 2>&1
FK_NCU_LAYER=1 timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -o gpurun_out/r02/headline_full -f python bench.py --no-cpu-baseline --no-e2e --no-isolated --no-check \
  > gpurun_out/r02/headline_full.log 2>&1
ncu -i gpurun_out/r02/headline_full.ncu-rep --page raw --csv > gpurun_out/r02/headline_full_raw.csv 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r02/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
  --no-isolated --no-check > /dev/null 2>&1
tail -n 3 gpurun_out/r02/traffic_summary.txt
