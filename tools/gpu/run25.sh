mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none -k regex:"k_kip|k_moddown|k_modup" -s 5 -c 5 -o gpurun_out/prof_ks python tools/prof_rotate.py > gpurun_out/ncu25.log 2>&1; echo ncu=$?
timeout 300 ncu --nvtx --nvtx-include "ks.modup/" --metrics gpu__time_duration.sum --csv --log-file gpurun_out/nvtx_modup.csv python tools/prof_rotate.py > gpurun_out/ncu25b.log 2>&1; echo nvtx=$?
