# Round-1 evidence run: parity, smoke, bench lines for every config, ncu launch list + full capture.
mkdir -p gpurun_out/ev
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/ev/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/ev/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/ev/smoke.log
timeout 600 python bench.py > gpurun_out/ev/bench_llama13b_p6000_b64.jsonl 2> gpurun_out/ev/bench.err
for c in llama13b_p6000_b128 llama13b_p6000_b256 llama7b_p6000_b64 mapreduce_13b nested_13b; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/ev/bench_$c.jsonl 2>> gpurun_out/ev/bench.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ev/bench_reference.jsonl 2>> gpurun_out/ev/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"fk_" -s 130 -c 130 --csv --log-file gpurun_out/ev/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ev/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fk_private|fk_prefix_tc|fk_merge" -s 60 -c 3 -o gpurun_out/ev/prof python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ev/ncu_full.log 2>&1
