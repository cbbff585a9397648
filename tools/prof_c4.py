"""Profiling driver: one compact layer (default C4 2048x2048, streamed W^T; `DxM` argument for another shape),
2 launches."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from bench import gen_compact  # noqa: E402
from paper_2509_09424_b200 import Context  # noqa: E402

ctx = Context(16, 12, 4, 3)
d, m = (int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "2048x2048").split("x"))
w = ctx.weights(synth.gen_W(5, d, m))
x = gen_compact(ctx, 3, d, 12)
y = torch.empty((m, ctx.wire_bytes(12)), dtype=torch.uint8, device="cuda")
for _ in range(2):
    ctx.pcmm_ternary_compact(x, w, y, level=12)
torch.cuda.synchronize()
