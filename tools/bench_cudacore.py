"""Time the CUDA-core Layout-A accumulate (opts.kernel = 1, accum.cu) on the C2 layer, uint64 words resident in HBM.
Prints one JSON line: ms per layer, term-words/s and the derived ALU-issue fraction (2 lane-ops per term-word)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from bench import time_loop  # noqa: E402
from paper_2509_09424_b200 import Context  # noqa: E402

ctx = Context(16, 12, 4, 3)
L, n, d, m = 12, ctx.n, 768, 768
W = synth.gen_W(synth.SEED_BASE + 102, d, m)
w = ctx.weights(W)
x = synth.gen_words_torch(synth.SEED_BASE + 2, ctx.q, d, L, n)
y = torch.empty((m, 2, L, n), dtype=torch.int64, device="cuda")
fn = lambda: ctx.pcmm_ternary(x, w, y, level=L, kernel=1)  # noqa: E731
for _ in range(2):
    fn()
ms = time_loop(fn, 5, torch.cuda.current_stream())
tw = int(np.count_nonzero(W)) * 2 * L * n
print(json.dumps({"ms": ms, "term_words_per_s": tw / (ms * 1e-3),
                  "alu_frac": 2 * tw / (ms * 1e-3) / (148 * 64 * 1.965e9)}))
