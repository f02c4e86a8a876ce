# co-run A/B + parity
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu3.log
for c in 0 1; do
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --corun $c > gpurun_out/bench3_corun$c.log 2>&1
done
for r in 60 100 130; do
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --prefix-rate-pct $r > gpurun_out/bench3_rate$r.log 2>&1
done
timeout 300 python profiles/step_gaps.py > gpurun_out/step_gaps3.log 2>&1
