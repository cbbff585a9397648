mkdir -p gpurun_out
for c in w6 w5 w5b mix; do timeout 120 python tools/gpu/dbg_tcc.py $c > gpurun_out/dbg_$c.log 2>&1; echo "$c rc=$?"; tail -1 gpurun_out/dbg_$c.log; done
timeout 900 python -m pytest tests/test_gpu_compact.py -x -q -p no:cacheprovider > gpurun_out/gpu_compact.log 2>&1; echo compact_tests=$?; tail -3 gpurun_out/gpu_compact.log
timeout 600 python tools/bench_compact.py --all > gpurun_out/compact.json 2> gpurun_out/compact.err; echo compact=$?; cat gpurun_out/compact.json
