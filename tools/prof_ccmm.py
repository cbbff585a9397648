"""Minimal driver for an ncu launch list of one CCMM output column at the Table III Q.K^T shape (C2 params)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
from paper_2509_09424_b200 import Context  # noqa: E402

cfg = synth.CONFIGS["C2"]
n, L, s, d, m = 1 << 16, 12, 2048, 96, 2048
ctx = Context(16, 12, 4, 3)
gal = lambda r: pow(5, r % (n // 2), 2 * n)
am = sorted(set([-(1 << u) for u in range(11)] + list(range(1, 64)) + [g * 64 for g in range(1, 32)]))
gs = [gal(r) for r in am]
ctx.load_keys(galois=gs, rot_keys=bench._random_keys(ctx, gs, cfg, n))
ctx.load_relin_key(bench._random_keys(ctx, [0], cfg, n)[0].contiguous())
a = synth.gen_words_torch(21, ctx.q, d, L, n)
src = synth.gen_words_torch(22, ctx.q, d, L, n)
mask = synth.gen_words_torch(23, ctx.q, 1, L, n)[0, 0].contiguous()
y = torch.empty((1, 2, L - 2, n), dtype=torch.int64, device="cuda")
for col in (65, 66):                      # first call warms up (scratch, tables); profile the second
    ctx.ccmm(a, src, mask, y, 1, s, d, m, L, col0=col, cols=1)
torch.cuda.synchronize()
print("ok")
