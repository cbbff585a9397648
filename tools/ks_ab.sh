# A/B timing of kernel variants (env switches read by libensi.so / alternative builds)
timeout 900 python -m pytest tests -m gpu -q -x -k "rotate or layout_b or n16 or rescale or ntt" 2>&1 | tail -1
bk() { timeout 300 python tools/bench_kernels.py --iters 20 --layout-b 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ntt_fwd']['us_per_limb'], d['ntt_inv']['us_per_limb'], d['rescale']['us_per_ct'], d['rotate_hoisted_32'], d['pcmm_layout_b_C2']['ms'])"; }
echo "== smem"; bk
cp tools/libensi_direct.so paper_2509_09424_b200/libensi.so
timeout 900 python -m pytest tests -m gpu -q -x -k "ntt" 2>&1 | tail -1
echo "== direct"; bk
