mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke21.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke21.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputests21.log 2>&1; echo tests=$?; tail -3 gpurun_out/gputests21.log
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/bench21.json 2> gpurun_out/bench21.err; echo bench=$?; tail -2 gpurun_out/bench21.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches21.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-rot --no-e2e > gpurun_out/ncu21a.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_accum_ternary -s 2 -c 1 -o gpurun_out/prof_cc python tools/bench_cudacore.py > gpurun_out/ncu21b.log 2>&1; echo ncu2=$?
