# diagnostics: step gaps, tcgen05 timeline, ncu full capture of the two attention kernels
mkdir -p gpurun_out
timeout 300 python profiles/step_gaps.py > gpurun_out/step_gaps.log 2>&1; echo "rc=$?" >> gpurun_out/step_gaps.log
sh profiles/build_tl.sh > gpurun_out/tl_build.log 2>&1 && FK_LIB_PATH=profiles/build/libforkattn_tl.so timeout 200 python profiles/tc_timeline.py > gpurun_out/tc_timeline.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fk_private|fk_prefix_tc|fk_merge" -s 30 -c 3 -o gpurun_out/prof_r1 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_full.log
