# variants of the compact accumulate's pipeline (timing only), each built in a scratch copy of the repo
mkdir -p gpurun_out
run() {  # name, nvcc extra flags
  v=$1; shift
  rm -rf /tmp/abl_$v && mkdir -p /tmp/abl_$v && cp -r paper_2509_09424_b200 synth.py bench.py oracle include tools tests /tmp/abl_$v/
  rm -f /tmp/abl_$v/paper_2509_09424_b200/libensi.so
  (cd /tmp/abl_$v && ENSI_NVCC_EXTRA="$*" python -c "from paper_2509_09424_b200 import build as b; b.build(force=True)" && timeout 300 python tools/bench_compact.py $ABL_ARGS) > gpurun_out/abl2_$v.json 2> gpurun_out/abl2_$v.err || echo "fail $v"
  echo "$v [$*] $(cat gpurun_out/abl2_$v.json)"
}
