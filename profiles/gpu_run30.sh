mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest30.log 2>&1; echo "rc=$?" >> gpurun_out/pytest30.log
timeout 300 python profiles/step_events.py > gpurun_out/step_events30.log 2>&1
sh profiles/build_tl.sh >/dev/null 2>&1; python profiles/cta_timeline.py > gpurun_out/cta_tl30.log 2>&1
for r in 50 70; do timeout 300 python bench.py --no-cpu-baseline --no-e2e --prefix-rate-pct $r > gpurun_out/bench30_r$r.log 2>&1; done
