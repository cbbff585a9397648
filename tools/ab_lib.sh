# A/B of the in-tree libensi.so against tools/libensi_abl.so: CUDA-core accumulate (kernel 1), parity first
cp paper_2509_09424_b200/libensi.so /tmp/base.so
cp tools/libensi_abl.so paper_2509_09424_b200/libensi.so
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "pcmm and 1" 2>&1 | tail -1
for i in 1 2; do
  cp /tmp/base.so paper_2509_09424_b200/libensi.so; echo -n "base "; timeout 300 python bench.py --no-cpu --no-e2e --no-rot --kernel 1 --steps 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'])"
  cp tools/libensi_abl.so paper_2509_09424_b200/libensi.so; echo -n "abl  "; timeout 300 python bench.py --no-cpu --no-e2e --no-rot --kernel 1 --steps 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'])"
done
cp /tmp/base.so paper_2509_09424_b200/libensi.so
