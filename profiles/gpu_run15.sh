mkdir -p gpurun_out
for r in 55 62 70 78; do timeout 300 python bench.py --no-cpu-baseline --no-e2e --prefix-rate-pct $r > gpurun_out/bench15_rate$r.log 2>&1; done
