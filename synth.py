"""Seeded synthetic inputs shared by tests/ and bench.py.

This module holds NONE of the method's arithmetic (no encoding, encryption, NTT or modular
accumulation).  It only draws data with the shapes and distributions of the paper's workloads
(DESIGN.md "Input recipe"):

* X ~ U[-1, 1] i.i.d. (s tokens x d features), as SPEC.md:251.
* W = BitNet b1.58 absmean quantisation of N(0,1) samples: W = RoundClip(w / mean|w|, -1, 1)
  (PAPER.md:239-240 BitLinear), giving P(0) ~ 0.31, P(+-1) ~ 0.345 each.
* uniform RNS words in [0, q_r) for timing-only repeats (the accumulate is data-oblivious).

The moduli are passed in by the caller; nothing here derives them.
"""
from __future__ import annotations

import numpy as np

SEED_BASE = 0x454E5349  # "ENSI"

# Configs C1..C5 of BASELINE.json.  log_n is log2 of the ring degree N'.
CONFIGS = {
    "C1": dict(log_n=12, L=3, alpha=1, dnum=3, s=16, shapes=[(16, 16)],
               desc="toy CKKS N'=2^12, 3 RNS limbs, 16x16 ternary PCMM"),
    "C2": dict(log_n=16, L=12, alpha=4, dnum=3, s=128, shapes=[(768, 768)],
               desc="N'=2^16, L=12, single 768x768 BitNet ternary PCMM"),
    "C3": dict(log_n=16, L=12, alpha=4, dnum=3, s=128, shapes=[(768, 3072), (3072, 768)],
               desc="N'=2^16, 768x3072 and 3072x768 FFN ternary PCMM, 128 tokens"),
    "C4": dict(log_n=16, L=12, alpha=4, dnum=3, s=512, shapes=[(2048, 2048)] * 4,
               desc="N'=2^16, 2048x2048 attention projections (Q,K,V,O), 512 tokens"),
    "C5": dict(log_n=16, L=12, alpha=4, dnum=3, s=512,
               shapes=[(2048, 6144), (2048, 2048), (2048, 5504), (2048, 5504), (5504, 2048)],
               desc="N'=2^16 block sweep at hidden 2048: QKV fused, O, gate, up, down (f=5504)"),
}


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def gen_X(seed: int, s: int, d: int) -> np.ndarray:
    """Activation matrix X (s x d), U[-1, 1]."""
    return rng(seed).uniform(-1.0, 1.0, size=(s, d))


def gen_W(seed: int, d: int, m: int) -> np.ndarray:
    """Ternary BitLinear weight (d x m) int8: RoundClip(w / mean|w|, -1, 1), w ~ N(0,1)."""
    w = rng(seed).standard_normal((d, m))
    gamma = np.mean(np.abs(w))
    return np.clip(np.rint(w / gamma), -1, 1).astype(np.int8)


def gen_words(seed: int, moduli, count: int, level: int, n: int) -> np.ndarray:
    """count ciphertexts of uniform RNS words: [count][2][level][n] uint64, limb r uniform in [0, moduli[r])."""
    g = rng(seed)
    out = np.empty((count, 2, level, n), np.uint64)
    for r in range(level):
        out[:, :, r, :] = g.integers(0, int(moduli[r]), size=(count, 2, n), dtype=np.uint64)
    return out


def edge_W(kind: str, d: int, m: int, seed: int = 0) -> np.ndarray:
    """Edge fixtures: zero, plus, minus, identity, neg_identity, permutation, toy."""
    if kind == "zero":
        return np.zeros((d, m), np.int8)
    if kind == "plus":
        return np.ones((d, m), np.int8)
    if kind == "minus":
        return -np.ones((d, m), np.int8)
    if kind == "identity":
        return np.eye(d, m, dtype=np.int8)
    if kind == "neg_identity":
        return -np.eye(d, m, dtype=np.int8)
    if kind == "permutation":
        assert d == m
        P = np.zeros((d, m), np.int8)
        P[np.arange(d), rng(seed).permutation(m)] = 1
        return P
    if kind == "toy":
        return np.array([[1, -1], [0, 1], [-1, 0], [0, 1]], np.int8)
    raise ValueError(kind)


def gen_words_torch(seed: int, moduli, count: int, level: int, n: int, device="cuda"):
    """Device-resident uniform RNS words (timing-only inputs): torch int64 [count][2][level][n], limb r in [0, q_r)."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    t = torch.empty((count, 2, level, n), dtype=torch.int64, device=device)
    for r in range(level):
        t[:, :, r, :].random_(0, int(moduli[r]), generator=g)
    return t
