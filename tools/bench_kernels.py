"""Per-primitive timings on the B200 at C2 parameters (N'=2^16, L=12, alpha=4, dnum=3): NTT/INTT, rescale,
hoisted rotations, Layout-B PCMM.  Timing-only inputs (uniform words, random keys: every kernel is
data-oblivious).  Prints one JSON object.  Usage: python tools/bench_kernels.py [--iters N] [--layout-b]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2509_09424_b200 import Context  # noqa: E402


def timed(fn, iters, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def random_keys(ctx, gs, dnum, T, n):
    keys = torch.empty((len(gs), dnum, 2, T, n), dtype=torch.int64, device="cuda")
    g = torch.Generator(device="cuda")
    g.manual_seed(7)
    for r in range(T):
        keys[:, :, :, r, :].random_(0, ctx.moduli[r], generator=g)
    return keys


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--layout-b", action="store_true")
    args = ap.parse_args()
    cfg = synth.CONFIGS["C2"]
    L, A, dnum, n = cfg["L"], cfg["alpha"], cfg["dnum"], 1 << cfg["log_n"]
    T = L + A
    ctx = Context(cfg["log_n"], L, A, dnum)
    out = {}
    rows = 768
    data = torch.empty((rows, n), dtype=torch.int64, device="cuda")
    for r in range(rows):
        pass
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    for lim in range(T):
        data[lim::T].random_(0, ctx.moduli[lim], generator=g)
    limbs = list(range(T))
    bytes_pass = rows * n * 8 * 2
    ms = timed(lambda: ctx.ntt(data, limbs), args.iters)
    out["ntt_fwd"] = {"rows": rows, "ms": ms, "us_per_limb": 1e3 * ms / rows,
                      "GBps_two_passes": 2 * bytes_pass / (ms * 1e-3) / 1e9}
    ms = timed(lambda: ctx.ntt(data, limbs, inverse=True), args.iters)
    out["ntt_inv"] = {"rows": rows, "ms": ms, "us_per_limb": 1e3 * ms / rows,
                      "GBps_two_passes": 2 * bytes_pass / (ms * 1e-3) / 1e9}
    # rescale 64 ciphertexts
    x = synth.gen_words_torch(5, ctx.q, 64, L, n)
    y = torch.empty((64, 2, L - 1, n), dtype=torch.int64, device="cuda")
    ms = timed(lambda: ctx.rescale(x, y, L), args.iters)
    out["rescale"] = {"cts": 64, "ms": ms, "us_per_ct": 1e3 * ms / 64}
    # hoisted rotations
    for batch in (1, 32, 128):
        gs = [pow(5, 128 * (b + 1), 2 * n) for b in range(batch)]
        keys = random_keys(ctx, gs, dnum, T, n)
        ctx.load_keys(galois=gs, rot_keys=keys)
        xr = synth.gen_words_torch(11, ctx.q, 1, L, n)
        yr = torch.empty((batch, 2, L, n), dtype=torch.int64, device="cuda")
        ms = timed(lambda: ctx.rotate_hoisted(xr, gs, yr, L), args.iters)
        out[f"rotate_hoisted_{batch}"] = {"ms": ms, "rot_per_s": batch / (ms * 1e-3)}
        del keys
    if args.layout_b:
        s, d, m = 128, 768, 768
        k = (n // 2) // s
        n_in = -(-d // k)
        gs = [pow(5, s * b, 2 * n) for b in range(1, k)]
        keys = random_keys(ctx, gs, dnum, T, n)
        ctx.load_keys(galois=gs, rot_keys=keys)
        W = synth.gen_W(synth.SEED_BASE + 102, d, m)
        w = ctx.weights(W)
        xb = synth.gen_words_torch(13, ctx.q, n_in, L, n)
        yb = torch.empty((m, 2, L, n), dtype=torch.int64, device="cuda")
        ms = timed(lambda: ctx.pcmm_ternary(xb, w, yb, level=L, layout=1, block_s=s), max(1, args.iters // 2), warm=1)
        out["pcmm_layout_b_C2"] = {"ms": ms, "rotations": (k - 1) * n_in, "s": s, "k": k, "n_in": n_in}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
