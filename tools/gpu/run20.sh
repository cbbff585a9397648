mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -k "kernel or wide or small_modulus or long_sum or sampled_columns or wire" > gpurun_out/t20.log 2>&1; echo tests=$?; tail -3 gpurun_out/t20.log
timeout 300 python tools/bench_cudacore.py; timeout 300 python tools/bench_compact.py
