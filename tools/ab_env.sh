# A/B timing of an env switch: bash tools/ab_env.sh VAR=value
timeout 900 python -m pytest tests -m gpu -q -x -k "rotate or layout_b or n16" 2>&1 | tail -1
bk() { timeout 300 python tools/bench_kernels.py --iters 10 --layout-b 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['rotate_hoisted_32']['rot_per_s'], d['rotate_hoisted_128']['rot_per_s'], d['pcmm_layout_b_C2']['ms'])"; }
for i in 1 2; do echo -n "default "; bk; echo -n "$1 "; env $1 bash -c "$(declare -f bk); bk"; done
