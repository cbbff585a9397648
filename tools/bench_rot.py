"""Rotation rates at C2 parameters (hoisted 128 / 32 per ModUp, 96 independent inputs) + Layout B; one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from bench import _random_keys, time_loop  # noqa: E402
from paper_2509_09424_b200 import Context  # noqa: E402

cfg = synth.CONFIGS["C2"]
L, A, dnum, n, s = cfg["L"], cfg["alpha"], cfg["dnum"], 1 << cfg["log_n"], cfg["s"]
ctx = Context(cfg["log_n"], L, A, dnum)
st = torch.cuda.current_stream()
out = {}
rows = 768
data = torch.empty((rows, n), dtype=torch.int64, device="cuda")
for lim in range(L + A):
    data[lim::L + A].random_(0, ctx.moduli[lim])
for name, inv in (("ntt_fwd_us", False), ("ntt_inv_us", True)):
    for _ in range(3):
        ctx.ntt(data, list(range(L + A)), inverse=inv)
    out[name] = 1e3 * time_loop(lambda: ctx.ntt(data, list(range(L + A)), inverse=inv), 20, st) / rows
del data
x = synth.gen_words_torch(11, ctx.q, 1, L, n)
for batch in (128, 32):
    gs = [pow(5, s * (b + 1), 2 * n) for b in range(batch)]
    ctx.load_keys(galois=gs, rot_keys=_random_keys(ctx, gs, cfg, n))
    y = torch.empty((batch, 2, L, n), dtype=torch.int64, device="cuda")
    for _ in range(2):
        ctx.rotate_hoisted(x, gs, y, L)
    out[f"hoisted_{batch}"] = batch / (1e-3 * time_loop(lambda: ctx.rotate_hoisted(x, gs, y, L), 8, st))
    del y
gs1 = [pow(5, s, 2 * n)]
ctx.load_keys(galois=gs1, rot_keys=_random_keys(ctx, gs1, cfg, n))
xb = synth.gen_words_torch(12, ctx.q, 96, L, n)
yb = torch.empty((96, 2, L, n), dtype=torch.int64, device="cuda")
for _ in range(2):
    ctx.rotate_batch(xb, gs1, yb, L)
out["independent"] = 96 / (1e-3 * time_loop(lambda: ctx.rotate_batch(xb, gs1, yb, L), 8, st))
print(json.dumps(out))
