mkdir -p gpurun_out
timeout 300 python profiles/step_events.py --opt PREFIX_RATE_PCT=50 > gpurun_out/step_events9.log 2>&1
for r in 35 45 60; do timeout 300 python bench.py --no-cpu-baseline --no-e2e --prefix-rate-pct $r > gpurun_out/bench9_rate$r.log 2>&1; done
