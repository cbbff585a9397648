mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke17.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke17.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputests17.log 2>&1; echo tests=$?; tail -3 gpurun_out/gputests17.log
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/bench17.json 2> gpurun_out/bench17.err; echo bench=$?; tail -2 gpurun_out/bench17.err
