# A/B of accumulate variants on the C2 headline (bench.py), alternating to cancel drift
#timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -k "pcmm or c2_" 2>&1 | tail -1
for i in 1 2; do
  for v in "ENSI_TC_FILL=80" "ENSI_TC_FILL=60" "ENSI_TC_FILL=40" "ENSI_TC_FILL=0"; do
    echo -n "[$v] "; env $v timeout 300 python bench.py --no-cpu --no-e2e --no-rot --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['gpu_launches'], {k: round(v['ms_per_layer'],2) for k, v in d['secondary']['layout_a_shapes'].items()} if 'layout_a_shapes' in d.get('secondary', {}) else '')"
  done
done
