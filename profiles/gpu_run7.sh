mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu7.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu7.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e --corun 0 > gpurun_out/bench7_c0.log 2>&1
for r in 50 80 110; do timeout 300 python bench.py --no-cpu-baseline --no-e2e --prefix-rate-pct $r > gpurun_out/bench7_rate$r.log 2>&1; done
timeout 300 python profiles/step_gaps.py --opt CORUN=0 > gpurun_out/step_gaps7_serial.log 2>&1
sh profiles/build_tl.sh > gpurun_out/tl_build.log 2>&1 && FK_LIB_PATH=profiles/build/libforkattn_tl.so timeout 200 python profiles/tc_timeline.py > gpurun_out/tc_timeline7.log 2>&1
