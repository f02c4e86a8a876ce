mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest26.log 2>&1; echo "rc=$?" >> gpurun_out/pytest26.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke26.log 2>&1; echo "rc=$?" >> gpurun_out/smoke26.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "tiny or fill_with or migration or host_tensor or nested or ragged" > gpurun_out/memcheck26.log 2>&1; echo "rc=$?" >> gpurun_out/memcheck26.log
timeout 600 python bench.py > gpurun_out/bench26.log 2>&1
