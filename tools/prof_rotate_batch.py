"""Profiling driver: 96 independent ciphertexts x 1 Galois element (ensi_rotate_batch) at C2 parameters, x3."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2509_09424_b200 import Context  # noqa: E402

cfg = synth.CONFIGS["C2"]
L, A, dnum, n = cfg["L"], cfg["alpha"], cfg["dnum"], 1 << 16
ctx = Context(16, L, A, dnum)
T = L + A
gs = [pow(5, 128, 2 * n)]
keys = torch.empty((1, dnum, 2, T, n), dtype=torch.int64, device="cuda")
for r in range(T):
    keys[:, :, :, r, :].random_(0, ctx.moduli[r])
ctx.load_keys(galois=gs, rot_keys=keys)
x = synth.gen_words_torch(12, ctx.q, 96, L, n)
y = torch.empty((96, 2, L, n), dtype=torch.int64, device="cuda")
for _ in range(3):
    ctx.rotate_batch(x, gs, y, L)
torch.cuda.synchronize()
