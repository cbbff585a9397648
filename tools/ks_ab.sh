# A/B timing of the key-switching kernel variants (env switches read by libensi.so)
timeout 900 python -m pytest tests -m gpu -q -x -k "rotate or layout_b or n16 or rescale or ntt" 2>&1 | tail -1
ENSI_KIP=inthint timeout 900 python -m pytest tests -m gpu -q -x -k "rotate or layout_b or n16" 2>&1 | tail -1
for v in "" "ENSI_KIP=inthint" "ENSI_KIP=fphint"; do echo "== $v"; env $v timeout 300 python tools/bench_kernels.py --iters 20 --layout-b 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['rotate_hoisted_32'], d['pcmm_layout_b_C2']['ms'])"; done
