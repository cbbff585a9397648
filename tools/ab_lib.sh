# A/B timing of tools/libensi_abl.so (an ablation / alternative build) against the in-tree build
bk() { timeout 300 python tools/bench_kernels.py --iters 20 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ntt_fwd']['us_per_limb'], d['ntt_inv']['us_per_limb'], d['rescale']['us_per_ct'], d['rotate_hoisted_128']['rot_per_s'])"; }
cp paper_2509_09424_b200/libensi.so /tmp/base.so
for i in 1 2; do
  cp /tmp/base.so paper_2509_09424_b200/libensi.so; echo -n "base "; bk
  cp tools/libensi_abl.so paper_2509_09424_b200/libensi.so; echo -n "abl  "; bk
done
cp /tmp/base.so paper_2509_09424_b200/libensi.so
