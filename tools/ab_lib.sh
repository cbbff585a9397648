# A/B of the in-tree libensi.so against tools/libensi_abl.so: NTT / rotation / rescale / Layout B (alternating)
cp paper_2509_09424_b200/libensi.so /tmp/base.so
bk() { timeout 300 python tools/bench_kernels.py --iters 20 --layout-b 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ntt_fwd']['us_per_limb'],4), round(d['ntt_inv']['us_per_limb'],4), round(d['rescale']['us_per_ct'],2), round(d['rotate_hoisted_128']['rot_per_s']), round(d['pcmm_layout_b_C2']['ms'],2))"; }
for i in 1 2; do
  cp /tmp/base.so paper_2509_09424_b200/libensi.so; echo -n "base "; bk
  cp tools/libensi_abl.so paper_2509_09424_b200/libensi.so; echo -n "abl  "; bk
done
cp /tmp/base.so paper_2509_09424_b200/libensi.so
