import os, sys, json
sys.path.insert(0, os.getcwd())
import torch, synth
from bench import _random_keys, time_loop, layout_b_plan
from paper_2509_09424_b200 import Context
cfg = synth.CONFIGS["C2"]; L, n, s = 12, 1 << 16, 128
ctx = Context(16, 12, 4, 3); st = torch.cuda.current_stream(); out = {}
for name, (dd, mm, bb) in (("C2_B64", (768, 768, 64)), ("C2_B32", (768, 768, 32))):
    kk, nin, B, G, rots = layout_b_plan(n, s, dd, mm, bb)
    gkb = sorted({pow(5, s * b, 2 * n) for b in range(1, B)} | {pow(5, s * B * g, 2 * n) for g in range(1, G)})
    ctx.load_keys(galois=gkb, rot_keys=_random_keys(ctx, gkb, cfg, n))
    w = ctx.weights(synth.gen_W(5, dd, mm)); xb = synth.gen_words_torch(14, ctx.q, nin, L, n)
    yb = torch.empty((mm, 2, L, n), dtype=torch.int64, device="cuda")
    row = {"G": G}
    for mode in (False, True):
        fn = lambda: ctx.pcmm_ternary(xb, w, yb, level=L, layout=1, block_s=s, baby=B, moddown_lazy=mode)
        fn(); row["lazy" if mode else "eager"] = time_loop(fn, 3, st)
    out[name] = row
    del xb, yb, w; torch.cuda.empty_cache()
print(json.dumps(out))
