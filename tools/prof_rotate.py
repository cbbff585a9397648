import sys, os
sys.path.insert(0, os.getcwd())
import torch, synth
from paper_2509_09424_b200 import Context
cfg = synth.CONFIGS["C2"]; L, A, dnum, n = cfg["L"], cfg["alpha"], cfg["dnum"], 1 << 16
ctx = Context(16, L, A, dnum); T = L + A
gs = [pow(5, 128 * (b + 1), 2 * n) for b in range(32)]
keys = torch.empty((32, dnum, 2, T, n), dtype=torch.int64, device="cuda")
for r in range(T): keys[:, :, :, r, :].random_(0, ctx.moduli[r])
ctx.load_keys(galois=gs, rot_keys=keys)
x = synth.gen_words_torch(11, ctx.q, 1, L, n)
y = torch.empty((32, 2, L, n), dtype=torch.int64, device="cuda")
for _ in range(3): ctx.rotate_hoisted(x, gs, y, L)
torch.cuda.synchronize()
