# A/B of key-switching build variants (timing only): bash tools/gpu/abl_ks.sh name "-DFLAG ..." [name flags ...]
mkdir -p gpurun_out
while [ $# -ge 2 ]; do
  v=$1; f=$2; shift 2
  rm -rf /tmp/ks_$v && mkdir -p /tmp/ks_$v && cp -r paper_2509_09424_b200 synth.py bench.py oracle include tools tests /tmp/ks_$v/
  rm -f /tmp/ks_$v/paper_2509_09424_b200/libensi.so
  (cd /tmp/ks_$v && ENSI_NVCC_EXTRA="$f" python -c "from paper_2509_09424_b200 import build as b; b.build(force=True)" && for i in 1 2; do timeout 300 python tools/bench_rot.py; done) > gpurun_out/ks_$v.json 2> gpurun_out/ks_$v.err || echo "fail $v"
  echo "$v [$f] $(cat gpurun_out/ks_$v.json | tr '\n' ' ')"
done
