"""Profiling driver: forward + inverse NTT over 768 rows at C2 parameters (N'=2^16), 3 times each."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2509_09424_b200 import Context  # noqa: E402

ctx = Context(16, 12, 4, 3)
T, n, rows = 16, 1 << 16, 768
data = torch.empty((rows, n), dtype=torch.int64, device="cuda")
for lim in range(T):
    data[lim::T].random_(0, ctx.moduli[lim])
for _ in range(3):
    ctx.ntt(data, list(range(T)))
    ctx.ntt(data, list(range(T)), inverse=True)
torch.cuda.synchronize()
