mkdir -p gpurun_out
for c in llama13b_p6000_b128 llama13b_p6000_b256 llama7b_p6000_b64 mapreduce_13b nested_13b; do timeout 400 python bench.py --no-cpu-baseline --no-e2e --config $c --steps 20 > gpurun_out/bench16_$c.log 2>&1; done
