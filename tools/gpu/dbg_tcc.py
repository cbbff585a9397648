"""Debug probe for the compact tensor-core accumulate: one case per process (an illegal instruction poisons the
context).  usage: python tools/gpu/dbg_tcc.py <case>"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch

import oracle
import synth
from paper_2509_09424_b200 import Context
from paper_2509_09424_b200.ensi import wire_pack_host, wire_unpack_host


def primes(m2n, below, count, skip=0):
    import sympy
    out, v = [], (below - 1) // m2n * m2n + 1
    while len(out) < count + skip:
        if v < below and sympy.isprime(v):
            out.append(v)
        v -= m2n
    return out[skip:]


def run(bits, d=16, m=16):
    m2n = 1 << 13
    q = [primes(m2n, 1 << b, 1, skip=i)[0] for i, b in enumerate(bits)]
    p = [primes(m2n, 1 << 59, 1)[0]]
    L = len(q)
    ctx = Context(12, L, 1, L, q=q, p=p)
    o = oracle.Oracle(12, L, 1, L, q=q, p=p)
    x = synth.gen_words(5, o.q, d, L, o.n)
    W = synth.gen_W(6, d, m)
    xc = torch.from_numpy(wire_pack_host(x, ctx.wire_widths(L))).cuda()
    yc = torch.zeros((m, ctx.wire_bytes(L)), dtype=torch.uint8, device="cuda")
    ctx.pcmm_ternary_compact(xc, ctx.weights(W), yc, level=L)
    torch.cuda.synchronize()
    got = wire_unpack_host(yc.cpu().numpy(), ctx.wire_widths(L), L, ctx.n)
    ok = (got == o.pcmm_a(x, W)).all()
    print("bits", bits, "d", d, "m", m, "ok", bool(ok), flush=True)


CASES = {"w8": [60], "w7": [55], "w6": [47], "w5": [40], "w5b": [34], "mix": [60, 47, 55, 34],
         "w8big": [60]}
if __name__ == "__main__":
    c = sys.argv[1]
    if c == "w8big":
        run(CASES[c], 300, 300)
    else:
        run(CASES[c])
