mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest19.log 2>&1; echo "rc=$?" >> gpurun_out/pytest19.log
for o in 0 1; do timeout 300 python profiles/step_events.py --opt LAUNCH_ORDER=$o > gpurun_out/step_events19_o$o.log 2>&1; done
timeout 300 python profiles/step_events.py --opt LAUNCH_ORDER=1 --opt PREFIX_RATE_PCT=65 > gpurun_out/step_events19_o1r65.log 2>&1
timeout 300 python profiles/step_gaps.py --opt LAUNCH_ORDER=1 > gpurun_out/step_gaps19.log 2>&1
