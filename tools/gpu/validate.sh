# Full GPU validation in one gpurun call: build + smoke, the -m gpu suite, one bench line, the headline launch list
# and an ncu --set full capture of the headline kernel.  Outputs under gpurun_out/.
#   gpurun --timeout 3600 -- 'bash tools/gpu/validate.sh'
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputests.log 2>&1; echo tests=$?; tail -2 gpurun_out/gputests.log
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu --no-rot --no-e2e > gpurun_out/ncu_launches.log 2>&1; echo launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_accum_tcc -s 3 -c 1 -o gpurun_out/prof_tcc \
    python bench.py --steps 1 --warmup 3 --no-cpu --no-rot --no-e2e > gpurun_out/ncu_tcc.log 2>&1; echo ncu=$?
