"""A/B timing of the Layout-A accumulate: uint64 words (k_accum_tc2) vs compact words (k_accum_tcc) at the BASELINE
shapes (C2 768x768 and the C3-C5 projections), device-resident inputs, CUDA events.  Prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2509_09424_b200 import Context  # noqa: E402


def t(fn, steps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / steps


def main():
    ctx = Context(16, 12, 4, 3)
    L, n = 12, ctx.n
    wb = ctx.wire_bytes(L)
    shapes = [(768, 768)] + ([(768, 3072), (3072, 768), (2048, 2048), (2048, 5504), (5504, 2048)]
                             if "--all" in sys.argv else [])
    out = {}
    for d, m in shapes:
        W = synth.gen_W(synth.SEED_BASE + d + m, d, m)
        w = ctx.weights(W)
        x = synth.gen_words_torch(17, ctx.q, d, L, n)
        y = torch.empty((m, 2, L, n), dtype=torch.int64, device="cuda")
        u64 = t(lambda: ctx.pcmm_ternary(x, w, y, level=L))
        xc = torch.empty((d, wb), dtype=torch.uint8, device="cuda")
        ctx.wire_pack(x, xc, L)
        del x, y
        torch.cuda.empty_cache()
        yc = torch.empty((m, wb), dtype=torch.uint8, device="cuda")
        cmp = t(lambda: ctx.pcmm_ternary_compact(xc, w, yc, level=L))
        byts = (d + m) * wb
        out[f"{d}x{m}"] = {"u64_ms": u64, "compact_ms": cmp, "compact_GBps": byts / cmp / 1e6,
                           "compact_hbm_frac": byts / cmp / 1e6 / 6454.3}
        del xc, yc, w
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
