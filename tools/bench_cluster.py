"""Timing of the compact accumulate per launch shape (opts.cluster_pairs = 0 auto, 1..4) at the BASELINE shapes:
calibrates accum_tcc.cu's kFeed cost model.  Device-resident compact inputs, CUDA events.  One JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2509_09424_b200 import Context  # noqa: E402


def t(fn, steps=6, warm=2):
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
    L = 12
    wb = ctx.wire_bytes(L)
    out = {}
    shapes = [(768, 768), (768, 3072), (3072, 768), (2048, 2048), (2048, 5504), (5504, 2048), (2048, 6144), (2048, 11008)]
    if len(sys.argv) > 1:
        shapes = [tuple(int(v) for v in a.split("x")) for a in sys.argv[1:]]
    for d, m in shapes:
        w = ctx.weights(synth.gen_W(synth.SEED_BASE + d + m, d, m))
        xc = torch.randint(0, 256, (d, wb), dtype=torch.uint8, device="cuda")   # timing only: any bytes
        yc = torch.empty((m, wb), dtype=torch.uint8, device="cuda")
        row = {}
        for cp in (0, 1, 2, 3, 4, 5, 6, 8):
            try:
                ms = t(lambda: ctx.pcmm_ternary_compact(xc, w, yc, level=L, cluster_pairs=cp))
            except Exception as ex:  # a cluster size that cannot be resident
                row[str(cp)] = str(ex)[:80]
                continue
            c, k = ctx.last_compact_plan()
            row[str(cp)] = {"ms": round(ms, 3), "c": c, "clusters": k, "sms": 2 * c * k}
        out[f"{d}x{m}"] = row
        print(json.dumps({f"{d}x{m}": row}), flush=True)
        del xc, yc, w
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
