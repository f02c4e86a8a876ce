mkdir -p gpurun_out
timeout 300 python profiles/step_events.py > gpurun_out/step_events10.log 2>&1
timeout 600 python bench.py > gpurun_out/bench10.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench10_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"fk_" -s 130 -c 130 --csv --log-file gpurun_out/launches10.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu10.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fk_private|fk_prefix_tc|fk_merge" -s 60 -c 3 -o gpurun_out/prof10 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full10.log 2>&1
