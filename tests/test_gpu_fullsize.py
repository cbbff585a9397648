"""Full-size (BASELINE.json configs[1], C2: N'=2^16, L=12, 768x768) parity in the launch configuration bench.py
times: sampled output columns compared word for word with the oracle, real pk-encryptions decrypted against
the float64 product (max-abs <= 1e-4), and full-size rotations / NTT / rescale bit-exact."""
import os

import numpy as np
import pytest

import oracle
import synth

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

DELTA = 2.0 ** 40
NTH = max(1, min(64, os.cpu_count() or 1))


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.fixture(scope="module")
def c2(torch_cuda):
    from paper_2509_09424_b200 import Context
    cfg = synth.CONFIGS["C2"]
    o = oracle.Oracle(cfg["log_n"], cfg["L"], cfg["alpha"], cfg["dnum"])
    skc, sk, pk = o.keygen(synth.SEED_BASE + 2)
    ctx = Context(cfg["log_n"], cfg["L"], cfg["alpha"], cfg["dnum"])
    ctx.load_keys(sk_ntt=sk)
    return o, sk, pk, ctx


def _dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).cuda()


@pytest.mark.parametrize("kernel", [2, 4, 3, 1])
def test_c2_sampled_columns_bit_exact(c2, torch_cuda, kernel):
    """768x768 on uniform words (data-oblivious accumulate): 3 full output columns == oracle Alg. 1."""
    o, sk, pk, ctx = c2
    torch = torch_cuda
    d = m = 768
    x = synth.gen_words(synth.SEED_BASE + 2, o.q, d, 12, o.n)
    W = synth.gen_W(synth.SEED_BASE + 102, d, m)
    xd = _dev(torch, x)
    yd = torch.empty((m, 2, 12, o.n), dtype=torch.int64, device="cuda")
    w = ctx.weights(W)
    ctx.pcmm_ternary(xd, w, yd, level=12, kernel=kernel)
    torch.cuda.synchronize()
    cols = [0, 377, 767]
    want = o.pcmm_a(x, W, cols=cols, nthreads=NTH)
    got = yd[cols].cpu().numpy().view(np.uint64)
    assert (got == want).all()
    # every output word is canonical (property at any size), checked on a strided sample of all outputs
    qv = torch.tensor(o.q, dtype=torch.int64, device="cuda").view(1, 1, 12, 1)
    assert bool((yd[:, :, :, ::97] >= 0).all()) and bool((yd[:, :, :, ::97] < qv).all())


def test_c2_encrypted_decrypts_to_product(c2, torch_cuda):
    """Real pk-encryptions of X (128 tokens x 768) -> PCMM -> decrypt == X.W within 1e-4 (north star)."""
    o, sk, pk, ctx = c2
    torch = torch_cuda
    s, d, m = 128, 768, 768
    X = synth.gen_X(synth.SEED_BASE + 2, s, d)
    W = synth.gen_W(synth.SEED_BASE + 102, d, m)
    m_res = np.stack([o.encode(X[:, j], 12, DELTA) for j in range(d)])
    x = o.encrypt_batch(np.arange(d, dtype=np.uint64) + np.uint64(123456), pk, 12, m_res, nthreads=NTH)
    del m_res
    xd = _dev(torch, x)
    yd = torch.empty((m, 2, 12, o.n), dtype=torch.int64, device="cuda")
    ctx.pcmm_ternary(xd, ctx.weights(W), yd, level=12)
    torch.cuda.synchronize()
    ref = X @ W.astype(np.float64)
    worst = 0.0
    for i in range(0, m, 37):
        z = ctx.decrypt_debug(yd, i, 12)
        worst = max(worst, float(np.max(np.abs(z[:s] - ref[:, i]))), float(np.max(np.abs(z[s:]))))
    assert worst < 1e-4
    # the oracle agrees on one column word for word
    want = o.pcmm_a(x, W, cols=[111], nthreads=NTH)
    assert (yd[111:112].cpu().numpy().view(np.uint64) == want).all()


def test_c2_rotations_bit_exact(c2, torch_cuda):
    o, sk, pk, ctx = c2
    torch = torch_cuda
    from paper_2509_09424_b200 import Context
    rctx = Context(16, 12, 4, 3)
    gs = [o.galois(128), o.galois(128 * 255)]
    keys = np.stack([o.rotkey(777 + i, g, sk) for i, g in enumerate(gs)])
    rctx.load_keys(sk_ntt=sk, galois=gs, rot_keys=keys)
    z = np.random.default_rng(1).uniform(-1, 1, o.n // 2)
    ct = o.encrypt(5, pk, 12, o.encode(z, 12, DELTA))
    want = o.rotate_hoisted(ct, gs, keys)
    yd = torch.empty((2, 2, 12, o.n), dtype=torch.int64, device="cuda")
    rctx.rotate_hoisted(_dev(torch, ct[None]), gs, yd, 12)
    torch.cuda.synchronize()
    assert (yd.cpu().numpy().view(np.uint64) == want).all()
    got = rctx.decrypt_debug(yd, 0, 12)
    assert np.max(np.abs(got - np.roll(z, -128))) < 1e-5


def test_c2_rescale_bit_exact(c2, torch_cuda):
    o, sk, pk, ctx = c2
    torch = torch_cuda
    x = synth.gen_words(9, o.q, 2, 12, o.n)
    want = np.stack([o.rescale(x[c]) for c in range(2)])
    yd = torch.empty((2, 2, 11, o.n), dtype=torch.int64, device="cuda")
    ctx.rescale(_dev(torch, x), yd, 12)
    torch.cuda.synchronize()
    assert (yd.cpu().numpy().view(np.uint64) == want).all()


@pytest.mark.parametrize("d,m", [(768, 3072), (2048, 2048), (5504, 2048), (2048, 6144)])
def test_c3_c4_sampled_columns_bit_exact(c2, torch_cuda, d, m):
    """BASELINE configs[2] (768->3072, 8-CTA multicast clusters, resident W^T), configs[3] (2048x2048, streamed
    W^T) and configs[4]'s widest shapes (down 5504->2048: 43 streamed K blocks; fused Q/K/V 2048->6144) at full
    size: sampled output columns == oracle Alg. 1 word for word.  Inputs are seeded uniform
    words from synth (the accumulate is data-oblivious), copied to the host for the oracle."""
    o, sk, pk, ctx = c2
    torch = torch_cuda
    xd = synth.gen_words_torch(synth.SEED_BASE + 3, o.q, d, 12, o.n)
    W = synth.gen_W(synth.SEED_BASE + 103, d, m)
    yd = torch.empty((m, 2, 12, o.n), dtype=torch.int64, device="cuda")
    ctx.pcmm_ternary(xd, ctx.weights(W), yd, level=12)
    torch.cuda.synchronize()
    cols = [0, m // 2 + 5, m - 1]
    got = yd[cols].cpu().numpy().view(np.uint64)
    del yd
    x = xd.cpu().numpy().view(np.uint64)
    del xd
    want = o.pcmm_a(x, W, cols=cols, nthreads=NTH)
    assert (got == want).all()


@pytest.mark.parametrize("B", [0, 4])
def test_layout_b_full_ring_bit_exact(c2, torch_cuda, B):
    """Layout B at the C2 ring (N'=2^16, L=12, alpha=4, dnum=3) on real encryptions: 20 columns packed in blocks of
    s=2048 slots (k=16, n_in=2), hoisted baby steps (B = k, or B = 4 with giant steps) through the FP64 key
    switching -- every output word == the oracle's O11 schedule, block 0 decrypts to X.W."""
    o, sk, pk, ctx = c2
    torch = torch_cuda
    from paper_2509_09424_b200 import Context
    s, d, m = 2048, 20, 6
    k, n_in, Bq, G, rots = oracle.layout_b_plan(o.n, s, d, m, B)
    X = synth.gen_X(synth.SEED_BASE + 31, s, d) * 0.5
    W = synth.gen_W(synth.SEED_BASE + 131, d, m)
    slots = o.n // 2
    cts = []
    for c in range(n_in):
        zz = np.zeros(slots)
        for b in range(k):
            col = c * k + b
            if col < d:
                zz[b * s:(b + 1) * s] = X[:, col]
        cts.append(o.encrypt(5100 + c, pk, 12, o.encode(zz, 12, DELTA)))
    x = np.stack(cts)
    gk = oracle.layout_b_galois(o.n, o.log_n, s, Bq, G)
    keys = np.stack([o.rotkey(5200 + i, g, sk) for i, g in enumerate(gk)])
    want = o.pcmm_b(x, W, s, k, Bq, gk, keys)
    bctx = Context(16, 12, 4, 3)
    bctx.load_keys(sk_ntt=sk, galois=gk, rot_keys=keys)
    yd = torch.empty((m, 2, 12, o.n), dtype=torch.int64, device="cuda")
    bctx.pcmm_ternary(_dev(torch, x), W, yd, level=12, layout=1, block_s=s, baby=Bq)
    torch.cuda.synchronize()
    assert (yd.cpu().numpy().view(np.uint64) == want).all()
    ref = X @ W.astype(np.float64)
    for i in range(m):
        z = bctx.decrypt_debug(yd, i, 12)
        assert np.max(np.abs(z[:s] - ref[:, i])) < 1e-4


def _rotkeys_parallel(o, sk, gs, seed0):
    """Real rotation keys for many Galois elements, generated on all host cores (the oracle's C keygen releases the
    GIL under ctypes)."""
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(NTH) as ex:
        return np.stack(list(ex.map(lambda ig: o.rotkey(seed0 + ig[0], ig[1], sk), enumerate(gs))))


def test_c2_rotate_hoisted_128_elements(c2, torch_cuda):
    """The hoisted-rotations/s bench shape at C2 parameters: one ciphertext rotated by 128 Galois elements in one
    call (four key-switch batches of 32 on the two internal streams with their own scratch sets).  Keys are seeded
    uniform words (the key switch is data-oblivious); outputs 0, 31, 32, 63, 64, 127 (every batch edge, both
    streams) == the oracle's hoisted rotations word for word."""
    o, sk, pk, ctx = c2
    torch = torch_cuda
    from paper_2509_09424_b200 import Context
    gs = [o.galois(r) for r in range(1, 129)]
    keys = synth.gen_words_torch(synth.SEED_BASE + 40, o.moduli, 128 * 3, 16, o.n).view(128, 3, 2, 16, o.n)
    rctx = Context(16, 12, 4, 3)
    rctx.load_keys(galois=gs, rot_keys=keys)
    ct = synth.gen_words(synth.SEED_BASE + 41, o.q, 1, 12, o.n)
    yd = torch.empty((128, 2, 12, o.n), dtype=torch.int64, device="cuda")
    rctx.rotate_hoisted(_dev(torch, ct), gs, yd, 12)
    torch.cuda.synchronize()
    sel = [0, 31, 32, 63, 64, 127]
    got = yd[sel].cpu().numpy().view(np.uint64)
    del yd
    ksel = keys[sel].cpu().numpy().view(np.uint64)
    want = o.rotate_hoisted(ct[0], [gs[i] for i in sel], ksel)
    assert (got == want).all()


def test_layout_b_c2_bench_schedule(c2, torch_cuda):
    """Layout B exactly as bench.py times it (C2: s = 128 tokens, 768 -> 768, k = 256 columns per ciphertext,
    n_in = 3 inputs, B = 256 baby steps, G = 1: 765 hoisted rotations with 255 keys in 8 key-switch batches on the
    two internal streams) on real pk-encryptions: output columns 0, 383, 767 == the oracle's O11 schedule word for
    word, and block 0 decrypts to X.W within 1e-4."""
    o, sk, pk, ctx = c2
    torch = torch_cuda
    from paper_2509_09424_b200 import Context
    s, d, m = 128, 768, 768
    k, n_in, B, G, rots = oracle.layout_b_plan(o.n, s, d, m, 0)
    assert (k, n_in, B, G, rots) == (256, 3, 256, 1, 765)
    X = synth.gen_X(synth.SEED_BASE + 42, s, d) * 0.25
    W = synth.gen_W(synth.SEED_BASE + 142, d, m)
    slots = o.n // 2
    zs = np.zeros((n_in, slots))
    for c in range(n_in):
        for b in range(k):
            if c * k + b < d:
                zs[c, b * s:(b + 1) * s] = X[:, c * k + b]
    m_res = np.stack([o.encode(zs[c], 12, DELTA) for c in range(n_in)])
    x = o.encrypt_batch(np.arange(n_in, dtype=np.uint64) + np.uint64(4200), pk, 12, m_res)
    gk = oracle.layout_b_galois(o.n, o.log_n, s, B, G)
    keys = _rotkeys_parallel(o, sk, gk, 4300)
    bctx = Context(16, 12, 4, 3)
    bctx.load_keys(sk_ntt=sk, galois=gk, rot_keys=keys)
    yd = torch.empty((m, 2, 12, o.n), dtype=torch.int64, device="cuda")
    bctx.pcmm_ternary(_dev(torch, x), bctx.weights(W), yd, level=12, layout=1, block_s=s)
    torch.cuda.synchronize()
    cols = [0, 383, 767]
    got = yd[cols].cpu().numpy().view(np.uint64)
    ref = X @ W.astype(np.float64)
    for i in cols:
        z = bctx.decrypt_debug(yd, i, 12)
        assert np.max(np.abs(z[:s] - ref[:, i])) < 1e-4, i
    del yd
    want = o.pcmm_b(x, W, s, k, B, gk, keys, cols=cols, nthreads=NTH)
    assert (got == want).all()


@pytest.mark.parametrize("d,m,baby,cols", [(3072, 768, 0, [0, 500, 767]), (768, 768, 64, [5, 700])])
def test_layout_b_lazy_moddown_full_size(c2, torch_cuda, d, m, baby, cols):
    """R19 (moddown_lazy) at full size, C2 parameters: BASELINE configs[2]'s down projection
    3072 -> 768 on its default plan (k = 256, n_in = 12, B = 128, G = 2: 1524 baby + 768 giant rotations; with one
    giant rotation per output the lazy form IS the eager one, checked on every output word) and 768 -> 768 with
    B = 64 (G = 4: 189 baby + 2304 giant rotations, three giant steps summed over Q_l u P per output, 8 chunks of
    96 outputs split over the two internal streams).  Seeded uniform words and keys (the path is data-oblivious);
    sampled output columns == the oracle's lazy O11 word for word, and the eager form (both timed by bench.py's
    layout_b_lazy_moddown row) == the oracle's eager O11."""
    o, sk, pk, ctx = c2
    torch = torch_cuda
    from paper_2509_09424_b200 import Context
    s = 128
    k, n_in, B, G, rots = oracle.layout_b_plan(o.n, s, d, m, baby)
    gk = oracle.layout_b_galois(o.n, o.log_n, s, B, G)
    keys = synth.gen_words_torch(synth.SEED_BASE + 50 + d, o.moduli, len(gk) * 3, 16, o.n).view(len(gk), 3, 2, 16,
                                                                                                 o.n)
    x = synth.gen_words(synth.SEED_BASE + 51 + d, o.q, n_in, 12, o.n)
    W = synth.gen_W(synth.SEED_BASE + 52 + d, d, m)
    bctx = Context(16, 12, 4, 3)
    bctx.load_keys(galois=gk, rot_keys=keys)
    w = bctx.weights(W)
    yd = torch.empty((m, 2, 12, o.n), dtype=torch.int64, device="cuda")
    bctx.pcmm_ternary(_dev(torch, x), w, yd, level=12, layout=1, block_s=s, baby=B, moddown_lazy=True)
    torch.cuda.synchronize()
    got = yd[cols].cpu().numpy().view(np.uint64)
    ye = torch.empty_like(yd)
    bctx.pcmm_ternary(_dev(torch, x), w, ye, level=12, layout=1, block_s=s, baby=B)     # the eager form bench times
    torch.cuda.synchronize()
    if G <= 2:
        assert torch.equal(yd, ye)
    got_e = ye[cols].cpu().numpy().view(np.uint64)
    del ye
    del yd
    bctx.close()
    kh = keys.cpu().numpy().view(np.uint64)
    del keys
    torch.cuda.empty_cache()
    want = o.pcmm_b(x, W, s, k, B, gk, kh, cols=cols, nthreads=NTH, lazy=True)
    assert (got == want).all()
    if G > 2:
        assert (got_e == o.pcmm_b(x, W, s, k, B, gk, kh, cols=cols, nthreads=NTH)).all()


def test_c2_integer_ntt_and_keyswitch_wide_moduli(torch_cuda):
    """N' = 2^16 with moduli >= 2^50: the integer v2 NTT passes (not the FP64 ones) in both directions on extreme and
    random rows, then hoisted rotations and rescale through the integer key-switching kernels -- word for word."""
    import sympy
    from paper_2509_09424_b200 import Context
    torch = torch_cuda
    m2n = 1 << 17

    def primes(below, cnt, skip=0):
        out, v = [], (below - 1) // m2n * m2n + 1
        while len(out) < cnt + skip:
            if v < below and sympy.isprime(v):
                out.append(v)
            v -= m2n
        return out[skip:]
    q = primes(1 << 56, 1) + primes(1 << 51, 2)
    p = primes(1 << 59, 1)
    o = oracle.Oracle(16, 3, 1, 3, q=q, p=p)
    ctx = Context(16, 3, 1, 3, q=q, p=p)
    assert ctx.moduli == o.moduli
    rows, limbs = [], []
    for li in range(4):
        qq = o.moduli[li]
        for pat in (np.full(o.n, qq - 1, np.uint64), np.tile(np.array([0, qq - 1], np.uint64), o.n // 2),
                    synth.gen_words(500 + li, [qq], 1, 1, o.n)[0, 0, 0]):
            rows.append(pat)
            limbs.append(li)
    rows = np.stack(rows)
    t = _dev(torch, rows)
    ctx.ntt(t, limbs)
    torch.cuda.synchronize()
    assert (t.cpu().numpy().view(np.uint64) == np.stack([o.ntt(limbs[i], rows[i]) for i in range(len(rows))])).all()
    t = _dev(torch, rows)
    ctx.ntt(t, limbs, inverse=True)
    torch.cuda.synchronize()
    assert (t.cpu().numpy().view(np.uint64) == np.stack([o.intt(limbs[i], rows[i]) for i in range(len(rows))])).all()
    skc, sk, pk = o.keygen(4600)
    gs = [o.galois(5), o.galois(-1024)]
    keys = np.stack([o.rotkey(4700 + i, g, sk) for i, g in enumerate(gs)])
    ctx.load_keys(sk_ntt=sk, galois=gs, rot_keys=keys)
    ct = synth.gen_words(4800, o.q, 1, 3, o.n)
    yd = torch.empty((2, 2, 3, o.n), dtype=torch.int64, device="cuda")
    ctx.rotate_hoisted(_dev(torch, ct), gs, yd, 3)
    yr = torch.empty((1, 2, 2, o.n), dtype=torch.int64, device="cuda")
    ctx.rescale(_dev(torch, ct), yr, 3)
    torch.cuda.synchronize()
    assert (yd.cpu().numpy().view(np.uint64) == o.rotate_hoisted(ct[0], gs, keys)).all()
    assert (yr.cpu().numpy().view(np.uint64)[0] == o.rescale(ct[0])).all()
