mkdir -p gpurun_out
for c in w8 w7 w6 w5 w5b mix w8big; do timeout 120 python tools/gpu/dbg_tcc.py $c > gpurun_out/dbg_$c.log 2>&1; echo "$c rc=$?"; tail -1 gpurun_out/dbg_$c.log; done
timeout 300 compute-sanitizer --show-backtrace device python tools/gpu/dbg_tcc.py w5 > gpurun_out/san_w5.log 2>&1; echo san=$?
timeout 300 compute-sanitizer --show-backtrace device python tools/gpu/dbg_tcc.py w8 > gpurun_out/san_w8.log 2>&1; echo san=$?
