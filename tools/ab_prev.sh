# A/B of the in-tree libensi.so against tools/libensi_prev.so (the previous commit's build): rotation rows
bk() { timeout 300 python tools/bench_kernels.py --iters 20 --layout-b 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['rotate_hoisted_128']['rot_per_s']), round(d['pcmm_layout_b_C2']['ms'],2))"; }
bi() { timeout 300 python bench.py --no-cpu --no-e2e --no-layout-b --no-ccmm 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['rotations_per_sec']; print('indep', round(r['independent_inputs']['value']), 'r32', round(r['per_32_batch']['value']))"; }
cp paper_2509_09424_b200/libensi.so /tmp/new.so
for i in 1 2; do
  cp /tmp/new.so paper_2509_09424_b200/libensi.so; echo -n "new: "; bk; bi
  cp tools/libensi_prev.so paper_2509_09424_b200/libensi.so; echo -n "prev: "; bk; bi
done
cp /tmp/new.so paper_2509_09424_b200/libensi.so
