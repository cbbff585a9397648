mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "ntt or rotate or rescale or layout_b" > gpurun_out/t5.log 2>&1; echo tests=$?; tail -3 gpurun_out/t5.log
timeout 600 python tools/ab_ntt.py > gpurun_out/ab_ntt.json 2> gpurun_out/ab_ntt.err; echo ab=$?; cat gpurun_out/ab_ntt.json; tail -3 gpurun_out/ab_ntt.err
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -p no:cacheprovider -k "rotations_bit_exact or rescale" > gpurun_out/t5b.log 2>&1; echo full=$?; grep -E "Error|passed|failed" gpurun_out/t5b.log | tail -5
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -p no:cacheprovider -k "rescale" > gpurun_out/t5c.log 2>&1; echo full=$?; grep -E "Error|passed|failed" gpurun_out/t5c.log | tail -5
