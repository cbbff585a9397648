mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_compact.py -x -q -p no:cacheprovider > gpurun_out/t8.log 2>&1; echo compact=$?; tail -3 gpurun_out/t8.log
timeout 600 python tools/bench_compact.py --all > gpurun_out/compact8.json 2> gpurun_out/compact8.err; echo bc=$?; cat gpurun_out/compact8.json
