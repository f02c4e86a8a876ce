mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest14.log 2>&1; echo "rc=$?" >> gpurun_out/pytest14.log
timeout 300 python profiles/step_events.py > gpurun_out/step_events14.log 2>&1
timeout 300 python profiles/step_events.py --opt PDL=1 > gpurun_out/step_events14_pdl1.log 2>&1
timeout 300 python profiles/step_gaps.py > gpurun_out/step_gaps14.log 2>&1
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench14.log 2>&1
