source tools/gpu/abl_tcc2.sh
runc() { v=$1; shift
  rm -rf /tmp/c_$v && mkdir -p /tmp/c_$v && cp -r paper_2509_09424_b200 synth.py bench.py oracle include tools /tmp/c_$v/
  rm -f /tmp/c_$v/paper_2509_09424_b200/libensi.so
  (cd /tmp/c_$v && ENSI_NVCC_EXTRA="$*" python -c "from paper_2509_09424_b200 import build as b; b.build(force=True)" && timeout 300 python tools/bench_cudacore.py) > gpurun_out/cc_$v.json 2> gpurun_out/cc_$v.err || echo "fail $v"
  echo "$v [$*] $(cat gpurun_out/cc_$v.json)"
}
runc ap4 -DENSI_ACC_AP=4
runc ap2 -DENSI_ACC_AP=2
runc ap8 -DENSI_ACC_AP=8
