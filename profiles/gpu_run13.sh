mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest13.log 2>&1; echo "rc=$?" >> gpurun_out/pytest13.log
sh profiles/build_tl.sh >/dev/null 2>&1; python profiles/cta_timeline.py > gpurun_out/cta_tl13.log 2>&1; python profiles/cta_timeline.py --opt CORUN=0 > gpurun_out/cta_tl13_serial.log 2>&1
for r in 40 50 60; do timeout 300 python bench.py --no-cpu-baseline --no-e2e --prefix-rate-pct $r > gpurun_out/bench13_rate$r.log 2>&1; done
