# ablation builds of the compact accumulate (timing only), each in a scratch copy of the repo
set -e
mkdir -p gpurun_out
for v in NONE NOCOMBINE NOEPI; do
  rm -rf /tmp/abl_$v && mkdir -p /tmp/abl_$v && cp -r paper_2509_09424_b200 synth.py bench.py oracle include tools /tmp/abl_$v/
  rm -f /tmp/abl_$v/paper_2509_09424_b200/libensi.so
  if [ $v != NONE ]; then export ENSI_NVCC_EXTRA="-DENSI_ABL_$v"; else unset ENSI_NVCC_EXTRA; fi
  (cd /tmp/abl_$v && python -c "from paper_2509_09424_b200 import build as b; b.build(force=True)" && timeout 300 python tools/bench_compact.py $ABL_ARGS) > gpurun_out/abl_$v.json 2> gpurun_out/abl_$v.err || echo "fail $v"
  echo "$v $(cat gpurun_out/abl_$v.json)"
done
