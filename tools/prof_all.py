"""Profiling driver: one instance of every C2 key-switching / NTT / rescale kernel (timing-only inputs), for a single
`ncu --set full` capture of the whole secondary path.  Warm-up first (lazy tables), then one marked round."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2509_09424_b200 import Context  # noqa: E402

cfg = synth.CONFIGS["C2"]
L, A, dnum, n = cfg["L"], cfg["alpha"], cfg["dnum"], 1 << 16
T = L + A
ctx = Context(16, L, A, dnum)
gs = [pow(5, 128 * (b + 1), 2 * n) for b in range(32)]
keys = torch.empty((32, dnum, 2, T, n), dtype=torch.int64, device="cuda")
for r in range(T):
    keys[:, :, :, r, :].random_(0, ctx.moduli[r])
ctx.load_keys(galois=gs, rot_keys=keys)
x = synth.gen_words_torch(11, ctx.q, 1, L, n)
y = torch.empty((32, 2, L, n), dtype=torch.int64, device="cuda")
xr = synth.gen_words_torch(5, ctx.q, 64, L, n)
yr = torch.empty((64, 2, L - 1, n), dtype=torch.int64, device="cuda")
rows = torch.empty((768, n), dtype=torch.int64, device="cuda")
for lim in range(T):
    rows[lim::T].random_(0, ctx.moduli[lim])
for _ in range(2):
    ctx.rotate_hoisted(x, gs, y, L)
    ctx.rescale(xr, yr, L)
    ctx.ntt(rows, list(range(T)))
    ctx.ntt(rows, list(range(T)), inverse=True)
torch.cuda.synchronize()
