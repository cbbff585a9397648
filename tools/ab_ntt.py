"""A/B of the NTT launch form at C2 parameters: ENSI_NTT_FUSED=1 (both passes in one persistent launch, the
intermediate kept in L2) vs 0 (two launches); NTT/INTT over 768 rows, hoisted rotations (128 per ModUp) and 96
independent rotations.  Timing-only uniform words and random keys.  Prints one JSON line."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from bench import _random_keys, time_loop  # noqa: E402
from paper_2509_09424_b200 import Context  # noqa: E402


def run(fused: str):
    os.environ["ENSI_NTT_FUSED"] = fused
    cfg = synth.CONFIGS["C2"]
    L, A, dnum, n, s = cfg["L"], cfg["alpha"], cfg["dnum"], 1 << cfg["log_n"], cfg["s"]
    T = L + A
    ctx = Context(cfg["log_n"], L, A, dnum)
    st = torch.cuda.current_stream()
    res = {}
    rows = 768
    data = torch.empty((rows, n), dtype=torch.int64, device="cuda")
    for lim in range(T):
        data[lim::T].random_(0, ctx.moduli[lim])
    for name, inv in (("ntt_fwd_us_per_limb", False), ("ntt_inv_us_per_limb", True)):
        for _ in range(3):
            ctx.ntt(data, list(range(T)), inverse=inv)
        res[name] = 1e3 * time_loop(lambda: ctx.ntt(data, list(range(T)), inverse=inv), 20, st) / rows
        res[name.replace("us_per_limb", "hbm_frac")] = rows * n * 16 / (res[name] * 1e-6 * rows) / 1e9 / 6454.3
    del data
    x = synth.gen_words_torch(11, ctx.q, 1, L, n)
    gs = [pow(5, s * (b + 1), 2 * n) for b in range(128)]
    ctx.load_keys(galois=gs, rot_keys=_random_keys(ctx, gs, cfg, n))
    y = torch.empty((128, 2, L, n), dtype=torch.int64, device="cuda")
    for _ in range(2):
        ctx.rotate_hoisted(x, gs, y, L)
    res["hoisted_rot_per_s"] = 128 / (1e-3 * time_loop(lambda: ctx.rotate_hoisted(x, gs, y, L), 5, st))
    del y
    gs1 = [pow(5, s, 2 * n)]
    ctx.load_keys(galois=gs1, rot_keys=_random_keys(ctx, gs1, cfg, n))
    xb = synth.gen_words_torch(12, ctx.q, 96, L, n)
    yb = torch.empty((96, 2, L, n), dtype=torch.int64, device="cuda")
    for _ in range(2):
        ctx.rotate_batch(xb, gs1, yb, L)
    res["independent_rot_per_s"] = 96 / (1e-3 * time_loop(lambda: ctx.rotate_batch(xb, gs1, yb, L), 5, st))
    ctx.close()
    del xb, yb, x
    torch.cuda.empty_cache()
    return res


if __name__ == "__main__":
    print(json.dumps({"fused": run("1"), "two_launch": run("0")}))
