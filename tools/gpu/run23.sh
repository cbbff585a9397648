mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none -k regex:k_accum_tcc -s 1 -c 1 -o gpurun_out/prof_c4 python tools/prof_c4.py > gpurun_out/ncu23.log 2>&1; echo ncu=$?
