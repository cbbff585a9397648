# A/B timing of an env switch: bash tools/ab_env.sh VAR=value  (parity subset first)
timeout 900 python -m pytest tests -m gpu -q -x -k "ntt or rotate or layout_b or n16 or rescale or custom or graph" 2>&1 | tail -1
bk() { timeout 300 python tools/bench_kernels.py --iters 20 --layout-b 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ntt_fwd']['us_per_limb'],4), round(d['ntt_inv']['us_per_limb'],4), round(d['rescale']['us_per_ct'],2), round(d['rotate_hoisted_128']['rot_per_s']), round(d['pcmm_layout_b_C2']['ms'],2))"; }
bi() { timeout 300 python bench.py --no-cpu --no-e2e --no-layout-b 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('indep', round(d['rotations_per_sec']['independent_inputs']['value']))"; }
for i in 1 2; do echo -n "default "; bk; bi; echo -n "$1 "; env $1 bash -c "$(declare -f bk); bk"; env $1 bash -c "$(declare -f bi); bi"; done
