mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "layout_b or ntt or pcmm_errors" > gpurun_out/t7a.log 2>&1; echo parity=$?; tail -3 gpurun_out/t7a.log
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -p no:cacheprovider -k "lazy" > gpurun_out/t7b.log 2>&1; echo full=$?; tail -3 gpurun_out/t7b.log
timeout 600 python -m pytest tests/test_gpu_dist.py tests/test_gpu_compact.py -q -p no:cacheprovider > gpurun_out/t7c.log 2>&1; echo dist=$?; tail -3 gpurun_out/t7c.log
bash tools/gpu/abl_tcc.sh
