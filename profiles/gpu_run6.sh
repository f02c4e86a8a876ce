mkdir -p gpurun_out
for r in 40 55 70; do timeout 300 python bench.py --no-cpu-baseline --no-e2e --prefix-rate-pct $r > gpurun_out/bench6_rate$r.log 2>&1; done
timeout 300 python profiles/step_gaps.py > gpurun_out/step_gaps6_corun.log 2>&1
timeout 300 python profiles/step_gaps.py --opt CORUN=0 > gpurun_out/step_gaps6_serial.log 2>&1
