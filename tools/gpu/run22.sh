mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_compact.py tests/test_gpu_dist.py -x -q -p no:cacheprovider > gpurun_out/t22.log 2>&1; echo compact=$?; tail -3 gpurun_out/t22.log; grep -E "^E " gpurun_out/t22.log | head -5
timeout 600 python tools/bench_compact.py --all > gpurun_out/compact22.json 2> gpurun_out/compact22.err; echo bc=$?; cat gpurun_out/compact22.json; tail -2 gpurun_out/compact22.err
