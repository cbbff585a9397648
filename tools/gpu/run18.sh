mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_compact.py -q -p no:cacheprovider > gpurun_out/t18.log 2>&1; echo dist=$?; tail -3 gpurun_out/t18.log
timeout 1200 python -m pytest tests/test_gpu_ccmm.py tests/test_gpu_compact.py tests/test_gpu_dist.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -k "not lazy" > gpurun_out/t18b.log 2>&1; echo seq=$?; tail -3 gpurun_out/t18b.log
