# A/B of the in-tree libensi.so against tools/libensi_abl.so on the C2 headline (alternating), after parity tests
cp paper_2509_09424_b200/libensi.so /tmp/base.so
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -k "pcmm or c2_ or c3_c4" 2>&1 | tail -1
for i in 1 2 3; do
  cp /tmp/base.so paper_2509_09424_b200/libensi.so
  echo -n "base "; timeout 300 python bench.py --no-cpu --no-e2e --no-rot --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], {k: round(v['ms_per_layer'],2) for k, v in d.get('secondary', {}).get('layout_a_shapes', {}).items()})"
  cp tools/libensi_abl.so paper_2509_09424_b200/libensi.so
  echo -n "abl  "; timeout 300 python bench.py --no-cpu --no-e2e --no-rot --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'])"
done
cp /tmp/base.so paper_2509_09424_b200/libensi.so
