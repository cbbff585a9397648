"""The fused gather epilogue on one GPU: the C2 compact layer stored into 1, 2 and 4 destination buffers (standing in
for 1, 2 and 4 GPUs' gathered buffers; on one GPU every extra destination is another 6.24 GB HBM write).  One JSON
line: ms per layer per destination count."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from bench import gen_compact, time_loop  # noqa: E402
from paper_2509_09424_b200 import Context  # noqa: E402

ctx = Context(16, 12, 4, 3)
d = m = 768
w = ctx.weights(synth.gen_W(synth.SEED_BASE + 102, d, m))
x = gen_compact(ctx, 3, d, 12)
wb = ctx.wire_bytes(12)
bufs = [torch.empty((m, wb), dtype=torch.uint8, device="cuda") for _ in range(4)]
st = torch.cuda.current_stream()
out = {}
for nd in (1, 2, 4):
    fn = lambda: ctx.pcmm_ternary_compact_gather(x, w, bufs[:nd], m, 0, 12)  # noqa: E731
    fn()
    out[f"{nd}_destinations_ms"] = time_loop(fn, 10, st)
fn = lambda: ctx.pcmm_ternary_compact(x, w, bufs[0], level=12)  # noqa: E731
fn()
out["plain_ms"] = time_loop(fn, 10, st)
print(json.dumps(out))
