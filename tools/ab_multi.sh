# A/B of several values of one env switch: bash tools/ab_multi.sh VAR v1 v2 ...  (parity subset with the first value)
var=$1; shift
env $var=$1 timeout 900 python -m pytest tests -m gpu -q -x -k "rotat or layout_b or ccmm or hoist or keyswitch" 2>&1 | tail -1
bk() { timeout 300 python tools/bench_kernels.py --iters 20 --layout-b 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['rotate_hoisted_128']['rot_per_s']), round(d['pcmm_layout_b_C2']['ms'],2))"; }
bi() { timeout 300 python bench.py --no-cpu --no-e2e --no-layout-b --no-ccmm 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['rotations_per_sec']; print('indep', round(r['independent_inputs']['value']), 'r32', round(r['per_32_batch']['value']))"; }
for i in 1 2; do
  echo -n "default: "; bk; bi
  for v in "$@"; do echo -n "$var=$v: "; env $var=$v bash -c "$(declare -f bk); bk"; env $var=$v bash -c "$(declare -f bi); bi"; done
done
