"""GPU parity for the CCMM path (R18) through the C ABI: the plaintext product,
Mult + relinearisation and the whole CCMM (both forms) against the oracle, every RNS word, and decryption against
the float64 matrix product.  C1 (N'=2^12, L=3) with real encryptions; N'=2^16 at the C2 prime chain on random
words (the key-switching, rescale and NTT kernels take their N'=2^16 FP64 paths there)."""
import numpy as np
import pytest

import oracle
import synth
from test_oracle_ccmm import _ccmm_setup

pytestmark = pytest.mark.gpu
DELTA = 2.0 ** 40


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).cuda()


def host(t):
    return t.cpu().numpy().view(np.uint64)


@pytest.fixture(scope="module")
def c1ctx(torch_cuda):
    from paper_2509_09424_b200 import Context
    o = oracle.Oracle(12, 3, 1, 3)
    skc, sk, pk = o.keygen(0x454E5349 + 1)
    ctx = Context(12, 3, 1, 3)
    ctx.load_keys(sk_ntt=sk)
    return o, sk, pk, ctx


def _load(ctx, keys, rlk):
    gs = list(keys.keys())
    ctx.load_keys(galois=gs, rot_keys=np.stack([keys[g] for g in gs]))
    ctx.load_relin_key(rlk)


def test_mul_plain_bit_exact(c1ctx, torch_cuda):
    o, sk, pk, ctx = c1ctx
    torch = torch_cuda
    x = synth.gen_words(501, o.q, 5, 3, o.n)
    pt = synth.gen_words(502, o.q, 1, 3, o.n)[0, 0]
    yd = torch.empty_like(dev(torch, x))
    sc = ctx.mul_plain(dev(torch, x), dev(torch, pt), yd, 3, 40.0, 40.0)
    torch.cuda.synchronize()
    got = host(yd)
    for c in range(5):
        assert (got[c] == o.mul_plain(x[c], pt)).all()
    assert sc == 80.0
    xd = dev(torch, x)                                   # in place (y == x) is allowed
    ctx.mul_plain(xd, dev(torch, pt), xd, 3)
    torch.cuda.synchronize()
    assert (host(xd) == got).all()


def test_mul_relin_bit_exact_and_decrypts(c1ctx, torch_cuda):
    o, sk, pk, ctx = c1ctx
    torch = torch_cuda
    rs = np.random.default_rng(503)
    xs, ys = rs.uniform(-1, 1, (3, o.n // 2)), rs.uniform(-1, 1, (3, o.n // 2))
    a = np.stack([o.encrypt(600 + c, pk, 3, o.encode(xs[c], 3, DELTA)) for c in range(3)])
    b = np.stack([o.encrypt(700 + c, pk, 3, o.encode(ys[c], 3, DELTA)) for c in range(3)])
    rlk = o.relinkey(504, sk)
    ctx.load_relin_key(rlk)
    yd = torch.empty((3, 2, 3, o.n), dtype=torch.int64, device="cuda")
    sc = ctx.mul_relin(dev(torch, a), dev(torch, b), yd, 3)
    torch.cuda.synchronize()
    got = host(yd)
    assert sc == 80.0
    for c in range(3):
        want = o.relin(o.mul_ct(a[c], b[c]), rlk)
        assert (got[c] == want).all()
        z = o.decrypt(sk, got[c], DELTA * DELTA)
        assert np.max(np.abs(z - xs[c] * ys[c])) < 1e-6


@pytest.mark.parametrize("form,s,d,m", [(2, 16, 4, 3), (2, 16, 3, 2), (2, 64, 16, 2), (2, 4, 1, 2), (2, 16, 11, 2), (2, 8, 8, 1),
                                        (1, 16, 4, 3), (1, 8, 2, 8), (1, 16, 3, 11)])
def test_ccmm_bit_exact_c1(c1ctx, torch_cuda, form, s, d, m):
    o, sk, pk, ctx = c1ctx
    torch = torch_cuda
    a, src, mask, keys, rlk, ref = _ccmm_setup(o, sk, pk, form, s, d, m, 900 + 10 * form + d)
    _load(ctx, keys, rlk)
    yd = torch.empty((m, 2, 1, o.n), dtype=torch.int64, device="cuda")
    sc = ctx.ccmm(dev(torch, a), dev(torch, src), dev(torch, mask), yd, form, s, d, m, 3)
    torch.cuda.synchronize()
    got = host(yd)
    want = o.ccmm(a, src, form, s, d, m, mask, keys, rlk)
    assert (got == want).all()
    assert abs(sc - (80.0 - np.log2(o.q[1]))) < 1e-9
    H = (o.n // 2) // s
    for i in range(m):
        z = o.decrypt(sk, got[i], 2.0 ** sc).reshape(H, s)
        assert np.max(np.abs(z - ref[:, :, i])) < 1e-4


def test_ccmm_column_range(c1ctx, torch_cuda):
    """A column shard [col0, col0 + cols) (one rank's share) equals those columns of the full product."""
    o, sk, pk, ctx = c1ctx
    torch = torch_cuda
    form, s, d, m = 1, 16, 3, 11
    a, src, mask, keys, rlk, ref = _ccmm_setup(o, sk, pk, form, s, d, m, 931)
    _load(ctx, keys, rlk)
    yd = torch.empty((4, 2, 1, o.n), dtype=torch.int64, device="cuda")
    ctx.ccmm(dev(torch, a), dev(torch, src), dev(torch, mask), yd, form, s, d, m, 3, col0=5, cols=4)
    torch.cuda.synchronize()
    want = o.ccmm(a, src, form, s, d, m, mask, keys, rlk, outputs=[5, 6, 7, 8])
    assert (host(yd) == want).all()


def test_ccmm_errors(c1ctx, torch_cuda):
    from paper_2509_09424_b200.ensi import EnsiError, ENSI_EDIM, ENSI_ELEVEL, ENSI_ENOKEY, ENSI_EINVAL
    o, sk, pk, ctx = c1ctx
    torch = torch_cuda
    a = torch.zeros((4, 2, 3, o.n), dtype=torch.int64, device="cuda")
    src = torch.zeros((2, 2, 3, o.n), dtype=torch.int64, device="cuda")
    mask = torch.zeros((3, o.n), dtype=torch.int64, device="cuda")
    y = torch.zeros((2, 2, 1, o.n), dtype=torch.int64, device="cuda")
    cases = [
        (dict(form=3, block_s=16, d=4, m=2), ENSI_EINVAL),
        (dict(form=2, block_s=12, d=4, m=2), ENSI_EDIM),
        (dict(form=2, block_s=2, d=4, m=2), ENSI_EDIM),      # d > s
        (dict(form=2, block_s=16, d=3, m=2), ENSI_EDIM),     # a.count != d
        (dict(form=1, block_s=16, d=4, m=2), ENSI_EDIM),     # src.count != d
        (dict(form=2, block_s=16, d=4, m=2, col0=2), ENSI_EDIM),
        (dict(form=2, block_s=16, d=4, m=2, col0=1, cols=2), ENSI_EDIM),
        (dict(form=2, block_s=16, d=4, m=2, col0=1, cols=1), ENSI_EDIM),   # y.count (2) != cols
    ]
    for kw, code in cases:
        with pytest.raises(EnsiError) as e:
            ctx.ccmm(a, src, mask, y, level=3, **kw)
        assert e.value.code == code, kw
    a2 = torch.zeros((4, 2, 2, o.n), dtype=torch.int64, device="cuda")
    with pytest.raises(EnsiError) as e:
        from paper_2509_09424_b200.ensi import CtView, CcmmOpts, lib
        import ctypes as C
        src2 = torch.zeros((2, 2, 2, o.n), dtype=torch.int64, device="cuda")
        av, sv = ctx.view(a2, 2), ctx.view(src2, 2)
        yv = CtView(y.data_ptr(), 2, 1, 40.0)
        ctx._check(lib().ensi_ccmm(ctx.h, C.byref(av), C.byref(sv), mask.data_ptr(), C.byref(yv),
                                   C.byref(CcmmOpts(2, 16, 4, 2, 0, 0)), None))
    assert e.value.code == ENSI_ELEVEL
    # rotation key missing: load keys without the alignment rotations
    ctx.load_keys(galois=[o.galois(-1)], rot_keys=np.zeros((1, 3, 2, 4, o.n), np.uint64))
    ctx.load_relin_key(np.zeros((3, 2, 4, o.n), np.uint64))
    with pytest.raises(EnsiError) as e:
        ctx.ccmm(a, src, mask, y, form=2, block_s=16, d=4, m=2, level=3)
    assert e.value.code == ENSI_ENOKEY


def test_ccmm_n16_c2_primes_bit_exact(torch_cuda):
    """N'=2^16 at the C2 prime chain (L=12, alpha=4, dnum=3), both forms, random words: the FP64 NTT, key
    switching (perm ModUp at level 12, plain at 11) and rescale paths."""
    from paper_2509_09424_b200 import Context
    torch = torch_cuda
    o = oracle.Oracle(16, 12, 4, 3)
    ctx = Context(16, 12, 4, 3)
    level = 12
    rs_keys = {}
    for form, s, d, m in [(2, 8, 2, 1), (1, 4, 2, 2)]:
        pi, amounts, _, _ = oracle.ccmm_plan(form, s, d, m)
        for r in amounts:
            g = o.galois(r)
            if g not in rs_keys:
                rs_keys[g] = synth.gen_words(8000 + len(rs_keys), o.moduli, 3, o.L + o.alpha, o.n)
    rlk = synth.gen_words(8100, o.moduli, 3, o.L + o.alpha, o.n)
    _load(ctx, rs_keys, rlk)
    for form, s, d, m in [(2, 8, 2, 1), (1, 4, 2, 2)]:
        a = synth.gen_words(8200 + form, o.q, d, level, o.n)
        src = synth.gen_words(8300 + form, o.q, m if form == 2 else d, level, o.n)
        mask = synth.gen_words(8400 + form, o.q, 1, level, o.n)[0, 0]
        yd = torch.empty((m, 2, level - 2, o.n), dtype=torch.int64, device="cuda")
        ctx.ccmm(dev(torch, a), dev(torch, src), dev(torch, mask), yd, form, s, d, m, level)
        torch.cuda.synchronize()
        want = o.ccmm(a, src, form, s, d, m, mask, rs_keys, rlk, outputs=[m - 1])
        assert (host(yd)[m - 1] == want[0]).all(), form


@pytest.mark.parametrize("level", [11, 9])
def test_rotation_partial_last_digit_n16(torch_cuda, level):
    """Key switching at a level alpha does not divide (C2 primes, alpha = 4: last digit of 3 / 1 limbs) -- the
    CCMM replicate steps run at level l - 1 = 11: hoisted and key-stationary batches vs the oracle, every word."""
    from paper_2509_09424_b200 import Context
    torch = torch_cuda
    o = oracle.Oracle(16, 12, 4, 3)
    ctx = Context(16, 12, 4, 3)
    gs = [o.galois(3), o.galois(-5)]
    keys = np.stack([synth.gen_words(8500 + i, o.moduli, 3, 16, o.n) for i in range(2)])
    ctx.load_keys(galois=gs, rot_keys=keys)
    x = synth.gen_words(8600 + level, o.q, 2, level, o.n)
    yh = torch.empty((2, 2, level, o.n), dtype=torch.int64, device="cuda")
    ctx.rotate_hoisted(dev(torch, x[:1]), gs, yh, level)
    yb = torch.empty((2, 2, level, o.n), dtype=torch.int64, device="cuda")
    ctx.rotate_batch(dev(torch, x), gs[1:], yb, level)
    torch.cuda.synchronize()
    assert (host(yh)[1] == o.rotate(x[0], gs[1], keys[1])).all()
    assert (host(yb)[1] == o.rotate(x[1], gs[1], keys[1])).all()


def test_integer_paths_large_moduli(torch_cuda):
    """Moduli >= 2^50 (up to just under 2^60) take the integer NTT, ModUp/KIP/ModDown and accumulate paths (no FP64
    shortcuts): PCMM, hoisted and batched rotations, Mult + relinearisation, rescale and a CCMM, word for word."""
    import sympy
    from paper_2509_09424_b200 import Context
    torch = torch_cuda
    m2n = 1 << 13

    def primes(below, cnt, skip=0):
        out, v = [], (below - 1) // m2n * m2n + 1
        while len(out) < cnt + skip:
            if sympy.isprime(v):
                out.append(v)
            v -= m2n
        return out[skip:]
    q = primes(1 << 60, 1) + primes(1 << 55, 2)
    p = primes(1 << 60, 1, skip=1)
    o = oracle.Oracle(12, 3, 1, 3, q=q, p=p)
    ctx = Context(12, 3, 1, 3, q=q, p=p)
    assert ctx.moduli == o.moduli
    skc, sk, pk = o.keygen(777)
    ctx.load_keys(sk_ntt=sk)
    # PCMM (Layout A)
    x = synth.gen_words(9500, o.q, 20, 3, o.n)
    W = synth.gen_W(9501, 20, 9)
    yd = torch.empty((9, 2, 3, o.n), dtype=torch.int64, device="cuda")
    ctx.pcmm_ternary(dev(torch, x), W, yd, level=3)
    torch.cuda.synchronize()
    assert (host(yd) == o.pcmm_a(x, W)).all()
    # rotations (hoisted and independent-input batches) and rescale
    gs = [o.galois(5), o.galois(-3)]
    keys = np.stack([o.rotkey(9600 + i, g, sk) for i, g in enumerate(gs)])
    ctx.load_keys(galois=gs, rot_keys=keys)
    ct = synth.gen_words(9602, o.q, 2, 3, o.n)
    yh = torch.empty((2, 2, 3, o.n), dtype=torch.int64, device="cuda")
    ctx.rotate_hoisted(dev(torch, ct[:1]), gs, yh, 3)
    yb = torch.empty((2, 2, 3, o.n), dtype=torch.int64, device="cuda")
    ctx.rotate_batch(dev(torch, ct), gs[1:], yb, 3)
    yr = torch.empty((2, 2, 2, o.n), dtype=torch.int64, device="cuda")
    ctx.rescale(dev(torch, ct), yr, 3)
    torch.cuda.synchronize()
    assert (host(yh) == o.rotate_hoisted(ct[0], gs, keys)).all()
    assert (host(yb)[1] == o.rotate(ct[1], gs[1], keys[1])).all()
    assert (host(yr)[0] == o.rescale(ct[0])).all()
    # Mult + relinearisation, then a CCMM (form 2) on real encryptions
    rlk = o.relinkey(9700, sk)
    ctx.load_relin_key(rlk)
    ym = torch.empty((1, 2, 3, o.n), dtype=torch.int64, device="cuda")
    ctx.mul_relin(dev(torch, ct[:1]), dev(torch, ct[1:]), ym, 3)
    torch.cuda.synchronize()
    assert (host(ym)[0] == o.relin(o.mul_ct(ct[0], ct[1]), rlk)).all()
    form, s, d, m = 2, 16, 3, 2
    a, src, mask, ckeys, crlk, ref = _ccmm_setup(o, sk, pk, form, s, d, m, 9800)
    _load(ctx, ckeys, crlk)
    yc = torch.empty((m, 2, 1, o.n), dtype=torch.int64, device="cuda")
    ctx.ccmm(dev(torch, a), dev(torch, src), dev(torch, mask), yc, form, s, d, m, 3)
    torch.cuda.synchronize()
    assert (host(yc) == o.ccmm(a, src, form, s, d, m, mask, ckeys, crlk)).all()


@pytest.mark.parametrize("form", [2, 1])
def test_ccmm_full_ring_decrypts(torch_cuda, form):
    """The full C2 ring (N'=2^16, L=12, 16 heads of s = 2048 tokens, real encryptions): CCMM output columns decrypt
    on the device (ensi_decrypt_debug) to the float64 products -- form 2 (A.B, d = 8) and form 1 (A.K^T with the
    Table III inner dimension 96 and m = 2048 keys' worth of alignment, sampled at columns 65 and 66: giant and baby
    steps)."""
    from paper_2509_09424_b200 import Context
    torch = torch_cuda
    o = oracle.Oracle(16, 12, 4, 3)
    skc, sk, pk = o.keygen(0x454E5349 + 2)
    ctx = Context(16, 12, 4, 3)
    ctx.load_keys(sk_ntt=sk)
    s, level = 2048, 12
    H = (o.n // 2) // s
    rs = np.random.default_rng(4400 + form)
    d, m, col0, cols = (8, 2, 0, 2) if form == 2 else (96, 2048, 65, 2)
    A = rs.uniform(-1, 1, (H, s, d))

    def enc(mat, sd):                      # mat [H][rows][ncols] -> one ciphertext per column
        Hh, rows, nc = mat.shape
        z = np.zeros((nc, o.n // 2))
        for h in range(Hh):
            z[:, h * s:h * s + rows] = mat[h].T
        m_res = np.stack([o.encode(v, level, DELTA) for v in z])
        return o.encrypt_batch(np.arange(nc, dtype=np.uint64) + np.uint64(sd), pk, level, m_res)
    a = enc(A, 100)
    if form == 2:
        Bm = rs.uniform(-1, 1, (H, d, m))
        src = enc(Bm, 200)
        ref = np.einsum("hsd,hdm->hsm", A, Bm)
    else:
        K = rs.uniform(-1, 1, (H, m, d))
        src = enc(K, 200)
        ref = np.einsum("hsd,hmd->hsm", A, K)
    pi, amounts, _, Ba = oracle.ccmm_plan(form, s, d, m)
    if form == 1:                          # only the keys the sampled columns use
        amounts = [r for r in amounts if r < 0] + [1, 2, Ba]
    z = np.zeros(o.n // 2)
    for h in range(H):
        z[h * s:h * s + s:pi] = 1.0
    coeffs = o.encode(z, level, float(o.q[level - 1]))
    mask = np.stack([o.ntt(i, coeffs[i]) for i in range(level)])
    gs = [o.galois(r) for r in amounts]
    ctx.load_keys(galois=gs, rot_keys=np.stack([o.rotkey(4500 + i, g, sk) for i, g in enumerate(gs)]))
    ctx.load_relin_key(o.relinkey(4600, sk))
    yd = torch.empty((cols, 2, level - 2, o.n), dtype=torch.int64, device="cuda")
    sc = ctx.ccmm(dev(torch, a), dev(torch, src), dev(torch, mask), yd, form, s, d, m, level, col0=col0, cols=cols)
    torch.cuda.synchronize()
    for c in range(cols):
        got = ctx.decrypt_debug(yd, c, level - 2, log2_scale=sc).reshape(H, s)
        err = np.max(np.abs(got - ref[:, :, col0 + c]))
        assert err < 1e-4, (form, c, err)


def test_mul_relin_many_pairs_split(c1ctx, torch_cuda):
    """Nine Mult + relinearisation pairs: the key switch of one element over >= 8 inputs runs split over the two
    internal streams -- still the oracle's words."""
    o, sk, pk, ctx = c1ctx
    torch = torch_cuda
    a = synth.gen_words(9900, o.q, 9, 3, o.n)
    b = synth.gen_words(9901, o.q, 9, 3, o.n)
    rlk = o.relinkey(9902, sk)
    ctx.load_relin_key(rlk)
    yd = torch.empty((9, 2, 3, o.n), dtype=torch.int64, device="cuda")
    ctx.mul_relin(dev(torch, a), dev(torch, b), yd, 3)
    torch.cuda.synchronize()
    got = host(yd)
    for c in (0, 4, 8):
        assert (got[c] == o.relin(o.mul_ct(a[c], b[c]), rlk)).all()
