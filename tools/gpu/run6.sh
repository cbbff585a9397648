mkdir -p gpurun_out
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r02a.json 2> gpurun_out/bench_r02a.err; echo bench=$?; tail -3 gpurun_out/bench_r02a.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_head.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-rot --no-e2e > gpurun_out/ncu_head.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_accum_tcc -s 1 -c 1 -o gpurun_out/prof_tcc python bench.py --steps 1 --warmup 1 --no-cpu --no-rot --no-e2e > gpurun_out/ncu_tcc.log 2>&1; echo ncu2=$?
ENSI_NTT_FUSED=1 timeout 600 ncu --set full --clock-control none -k regex:k_ntt_fused -s 2 -c 2 -o gpurun_out/prof_nttf python tools/prof_ntt.py > gpurun_out/ncu_nttf.log 2>&1; echo ncu3=$?
