"""The compact-layout tensor-core accumulate (ensi_pcmm_ternary_compact, accum_tcc.cu): ciphertexts resident in HBM as
ceil(bitlen(q_r)/8)-byte words.  Every output word == the oracle's Algorithm 1 (compared after the numpy host
deserialisation wire_unpack_host, which holds none of the method's arithmetic): real encryptions at C1, ragged
shapes and tail tiles, edge weights, every word width 5..8 bytes, the paper's N' = 2^14 ring, C2 full size in the
launch configuration bench.py times, and the host wire pipeline that now runs the compact kernel per slice."""
import os

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

DELTA = 2.0 ** 40
NTH = max(1, min(64, os.cpu_count() or 1))


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _compact_dev(torch, ctx, x, level):
    from paper_2509_09424_b200.ensi import wire_pack_host
    return torch.from_numpy(wire_pack_host(x, ctx.wire_widths(level))).cuda()


def _run(torch, ctx, x, W, level, kernel=0):
    from paper_2509_09424_b200.ensi import wire_unpack_host
    d, m = W.shape
    xc = _compact_dev(torch, ctx, x, level)
    yc = torch.full((m, ctx.wire_bytes(level)), 0xA5, dtype=torch.uint8, device="cuda")
    ctx.pcmm_ternary_compact(xc, ctx.weights(W), yc, level=level, kernel=kernel)
    torch.cuda.synchronize()
    return wire_unpack_host(yc.cpu().numpy(), ctx.wire_widths(level), level, ctx.n)


@pytest.fixture(scope="module")
def c1(torch_cuda):
    from paper_2509_09424_b200 import Context
    o = oracle.Oracle(12, 3, 1, 3)
    skc, sk, pk = o.keygen(synth.SEED_BASE + 1)
    ctx = Context(12, 3, 1, 3)
    ctx.load_keys(sk_ntt=sk)
    return o, sk, pk, ctx


def test_compact_c1_encrypted(c1, torch_cuda):
    """C1 (N' = 4096: 40-bit limbs in 85 tiles of 48 words + a 16-word tail, the 50-bit limb in 128 tiles of 32):
    16x16 on real pk-encryptions == oracle word for word, and decrypts to X.W."""
    o, sk, pk, ctx = c1
    torch = torch_cuda
    X = synth.gen_X(synth.SEED_BASE + 1, 16, 16)
    W = synth.gen_W(synth.SEED_BASE + 101, 16, 16)
    m_res = np.stack([o.encode(X[:, j], 3, DELTA) for j in range(16)])
    x = o.encrypt_batch(np.arange(16, dtype=np.uint64) + np.uint64(7000), pk, 3, m_res)
    got = _run(torch, ctx, x, W, 3)
    want = o.pcmm_a(x, W)
    assert (got == want).all()
    ref = X @ W.astype(np.float64)
    for i in (0, 7, 15):
        assert np.max(np.abs(o.decrypt(sk, got[i], DELTA)[:16] - ref[:, i])) < 1e-4


@pytest.mark.parametrize("d,m,level", [(37, 70, 3), (1, 1, 1), (130, 3, 3), (5, 300, 2), (900, 200, 1),
                                       (257, 513, 3)])
def test_compact_ragged(c1, torch_cuda, d, m, level):
    """Ragged d (K padding) and m (partial pair groups: single pairs for m <= 256, multicast clusters of 2 and 3
    pairs), levels 1..3, with words 0 and q - 1 at the tile edges."""
    o, sk, pk, ctx = c1
    torch = torch_cuda
    x = synth.gen_words(d * 1000 + m + 7, o.q, d, level, o.n)
    x[0, 0, 0, :7] = 0
    x[-1, 1, level - 1, :7] = np.uint64(o.q[level - 1] - 1)
    W = synth.gen_W(d + m + 7, d, m)
    assert (_run(torch, ctx, x, W, level) == o.pcmm_a(x, W, nthreads=4)).all()


@pytest.mark.parametrize("d,m,level", [(200, 1200, 3), (900, 3000, 2), (768, 3100, 1)])
def test_compact_every_cluster_shape(c1, torch_cuda, d, m, level):
    """The launch shape (opts.cluster_pairs = 1..4 and 8 CTA pairs per multicast cluster -- 16 CTAs is a non-portable
    cluster size -- and 0 = the per-layer choice):
    every co-resident cluster takes a contiguous run of (super-group, word tile) items, so runs cross super-groups
    (resident W^T reloaded mid-kernel: d <= 768) and super-groups overhang the padded W^T (5 / 12 / 13 pair groups
    in clusters of 2..4 pairs) -- the outputs are the same words as the oracle's Algorithm 1 for every shape.
    Resident (d = 200, 768) and streamed (d = 900) W^T."""
    from paper_2509_09424_b200.ensi import wire_unpack_host
    o, sk, pk, ctx = c1
    torch = torch_cuda
    x = synth.gen_words(d * 77 + m + level, o.q, d, level, o.n)
    W = synth.gen_W(d + 3 * m + level, d, m)
    cols = sorted({0, 1, 255, 256, 511, 767, 1023, 1200 - 1, m // 2, m - 257, m - 2, m - 1} & set(range(m)))
    want = o.pcmm_a(x, W, cols=cols, nthreads=NTH)
    xc = _compact_dev(torch, ctx, x, level)
    w = ctx.weights(W)
    shapes = set()
    from paper_2509_09424_b200.ensi import EnsiError, ENSI_ECUDA
    for cp in (0, 1, 2, 3, 4, 8):
        yc = torch.full((m, ctx.wire_bytes(level)), 0xA5, dtype=torch.uint8, device="cuda")
        try:
            ctx.pcmm_ternary_compact(xc, w, yc, level=level, cluster_pairs=cp)
        except EnsiError as ex:     # a non-portable 16-CTA cluster that this device cannot make resident
            assert cp == 8 and ex.code == ENSI_ECUDA
            continue
        torch.cuda.synchronize()
        c, k = ctx.last_compact_plan()
        assert 1 <= c <= 8 and k >= 1 and (cp == 0 or c == cp)
        shapes.add((c, k))
        got = wire_unpack_host(yc[cols].cpu().numpy(), ctx.wire_widths(level), level, ctx.n)
        assert (got == want).all(), (cp, c, k)
    assert len(shapes) >= 4


@pytest.mark.parametrize("kind", ["zero", "identity", "neg_identity", "permutation", "plus", "minus", "toy"])
def test_compact_edge_weights(c1, torch_cuda, kind):
    o, sk, pk, ctx = c1
    torch = torch_cuda
    d = m = 4 if kind == "toy" else 96
    if kind == "toy":
        m = 2
    W = synth.edge_W(kind, d, m, seed=5)
    x = synth.gen_words(78, o.q, d, 3, o.n)
    for r in range(3):
        x[:, :, r, 11:20] = np.uint64(o.q[r] - 1)
    assert (_run(torch, ctx, x, W, 3) == o.pcmm_a(x, W, nthreads=4)).all()


def test_compact_long_sum_all_q_minus_one(c1, torch_cuda):
    """d = 8300 terms of q - 1 (the largest |D| per byte plane): closed-form words (sum_j W_ji)(q - 1) mod q."""
    o, sk, pk, ctx = c1
    torch = torch_cuda
    d, m, level = 8300, 3, 2
    x = np.empty((d, 2, level, o.n), np.uint64)
    for r in range(level):
        x[:, :, r, :] = np.uint64(o.q[r] - 1)
    W = np.ones((d, m), np.int8)
    W[:, 1] = -1
    W[::3, 2] = -1
    got = _run(torch, ctx, x, W, level)
    for i in range(m):
        c = int(np.sum(W[:, i].astype(np.int64)))
        for r in range(level):
            assert (got[i, :, r] == np.uint64((c * (o.q[r] - 1)) % o.q[r])).all()


def _primes_1mod(mod2n, below, count, skip=0):
    import sympy
    out, v = [], (below - 1) // mod2n * mod2n + 1
    while len(out) < count + skip:
        if v < below and sympy.isprime(v):
            out.append(v)
        v -= mod2n
    return out[skip:]


def test_compact_every_word_width(torch_cuda):
    """User moduli with 5-, 6-, 7- and 8-byte words (2^33 .. 2^60): 6-byte limbs take 40-word tiles with an 8..32-word
    tail, 8-byte limbs 32-word tiles of 256 bytes -- every word == the oracle."""
    from paper_2509_09424_b200 import Context
    torch = torch_cuda
    m2n = 1 << 13
    q = [_primes_1mod(m2n, 1 << 60, 1)[0], _primes_1mod(m2n, 1 << 47, 1)[0], _primes_1mod(m2n, 1 << 55, 1)[0],
         _primes_1mod(m2n, 1 << 34, 1)[0]]
    p = [_primes_1mod(m2n, 1 << 60, 1, skip=1)[0]]
    ctx = Context(12, 4, 1, 4, q=q, p=p)
    assert [(v.bit_length() + 7) // 8 for v in q] == [8, 6, 7, 5]
    o = oracle.Oracle(12, 4, 1, 4, q=q, p=p)
    x = synth.gen_words(14700, o.q, 300, 4, o.n)
    for r in range(4):
        x[::7, :, r, ::5] = np.uint64(o.q[r] - 1)
    W = synth.gen_W(14701, 300, 260)
    assert (_run(torch, ctx, x, W, 4) == o.pcmm_a(x, W, nthreads=4)).all()


@pytest.mark.parametrize("L,alpha", [(12, 4), (48, 16)])
def test_compact_paper_ring_n14(torch_cuda, L, alpha):
    """N' = 2^14 (the paper's default ring) at l = 12 and 48: 96 slices per ciphertext (the tile table maximum)."""
    from paper_2509_09424_b200 import Context
    torch = torch_cuda
    o = oracle.Oracle(14, L, alpha, 3)
    ctx = Context(14, L, alpha, 3)
    x = synth.gen_words(14800 + L, o.q, 70, L, o.n)
    W = synth.gen_W(14801 + L, 70, 40)
    assert (_run(torch, ctx, x, W, L) == o.pcmm_a(x, W, nthreads=4)).all()


@pytest.mark.parametrize("log_n", [8, 13, 15])
def test_compact_other_rings(torch_cuda, log_n):
    """N' = 2^8 (the smallest compact ring: 5 full 48-word tiles and a 16-word tail per 40-bit slice), 2^13 and 2^15
    (32-word tails after 170 / 682 full tiles) at the C1 prime rule -- every word == the oracle."""
    from paper_2509_09424_b200 import Context
    torch = torch_cuda
    o = oracle.Oracle(log_n, 3, 1, 3)
    ctx = Context(log_n, 3, 1, 3)
    x = synth.gen_words(14900 + log_n, o.q, 140, 3, o.n)
    x[3, :, :, :9] = np.uint64(0)
    W = synth.gen_W(14901 + log_n, 140, 300)
    assert (_run(torch, ctx, x, W, 3) == o.pcmm_a(x, W, nthreads=4)).all()


def test_compact_c2_full_size_bench_launch(torch_cuda):
    """C2 (BASELINE configs[1]) exactly as bench.py times it: 768 compact input ciphertexts (8.1 MB each) -> 768
    outputs in one launch; three whole output columns == the oracle, and the uint64 tensor-core path agrees on
    every word of a strided sample of all outputs."""
    from paper_2509_09424_b200 import Context
    from paper_2509_09424_b200.ensi import wire_unpack_host
    torch = torch_cuda
    ctx = Context(16, 12, 4, 3)
    o = oracle.Oracle(16, 12, 4, 3)
    d = m = 768
    xd = synth.gen_words_torch(synth.SEED_BASE + 2, ctx.q, d, 12, ctx.n)
    W = synth.gen_W(synth.SEED_BASE + 102, d, m)
    w = ctx.weights(W)
    wb = ctx.wire_bytes(12)
    xc = torch.empty((d, wb), dtype=torch.uint8, device="cuda")
    ctx.wire_pack(xd, xc, 12)
    yc = torch.empty((m, wb), dtype=torch.uint8, device="cuda")
    ctx.pcmm_ternary_compact(xc, w, yc, level=12)
    y64 = torch.empty((m, 2, 12, ctx.n), dtype=torch.int64, device="cuda")
    ctx.pcmm_ternary(xd, w, y64, level=12)
    yu = torch.empty((m, 2, 12, ctx.n), dtype=torch.int64, device="cuda")
    ctx.wire_unpack(yc, yu, 12)
    torch.cuda.synchronize()
    assert bool((yu[:, :, :, ::61] == y64[:, :, :, ::61]).all())
    del yu, y64
    cols = [0, 400, 767]
    got = wire_unpack_host(yc[cols].cpu().numpy(), ctx.wire_widths(12), 12, ctx.n)
    x = xd.cpu().numpy().view(np.uint64)
    del xd, xc, yc
    assert (got == o.pcmm_a(x, W, cols=cols, nthreads=NTH)).all()


def test_compact_errors(c1, torch_cuda):
    from paper_2509_09424_b200.ensi import EnsiError, ENSI_EINVAL, ENSI_EDIM
    o, sk, pk, ctx = c1
    torch = torch_cuda
    wb = ctx.wire_bytes(3)
    w = ctx.weights(synth.gen_W(1, 4, 2))
    x = torch.zeros((4, wb), dtype=torch.uint8, device="cuda")
    y = torch.zeros((2, wb), dtype=torch.uint8, device="cuda")
    with pytest.raises(EnsiError) as e:
        ctx.pcmm_ternary_compact(x, w, y, level=3, kernel=1)
    assert e.value.code == ENSI_EINVAL
    with pytest.raises(EnsiError) as e:
        ctx.pcmm_ternary_compact(x[:3], w, y, level=3)
    assert e.value.code == ENSI_EDIM
    with pytest.raises(EnsiError) as e:
        ctx.pcmm_ternary_compact(x[:2], ctx.weights(synth.gen_W(2, 2, 2)), x[1:3], level=3)
    assert e.value.code == ENSI_EINVAL
    with pytest.raises(EnsiError) as e:
        ctx.pcmm_ternary_compact(x, w, y, level=3, cluster_pairs=9)
    assert e.value.code == ENSI_EINVAL


@pytest.mark.parametrize("d,m", [(768, 3072), (3072, 768), (2048, 2048), (2048, 5504), (5504, 2048), (2048, 6144)])
def test_compact_bench_shapes_sampled_columns(torch_cuda, d, m):
    """Every C3-C5 shape bench.py times on the compact layout (layout_a_shapes) at full size, in the launch
    configuration it times (one ensi_pcmm_ternary_compact call, the per-layer launch shape): 768->3072 (resident
    W^T, 12 pair groups), 3072->768 and 5504->2048 (streamed W^T, 24 / 43 K blocks), 2048^2, 2048->5504 and the fused
    Q/K/V 2048->6144 -- sampled output columns == the oracle's Algorithm 1, word for word."""
    from paper_2509_09424_b200 import Context
    from paper_2509_09424_b200.ensi import wire_unpack_host
    torch = torch_cuda
    ctx = Context(16, 12, 4, 3)
    o = oracle.Oracle(16, 12, 4, 3)
    xd = synth.gen_words_torch(synth.SEED_BASE + 5 + d, ctx.q, d, 12, ctx.n)
    W = synth.gen_W(synth.SEED_BASE + 6 + m, d, m)
    wb = ctx.wire_bytes(12)
    xc = torch.empty((d, wb), dtype=torch.uint8, device="cuda")
    ctx.wire_pack(xd, xc, 12)
    x = xd.cpu().numpy().view(np.uint64)
    del xd
    yc = torch.empty((m, wb), dtype=torch.uint8, device="cuda")
    ctx.pcmm_ternary_compact(xc, ctx.weights(W), yc, level=12)
    torch.cuda.synchronize()
    cols = [0, m // 2 + 7, m - 1]
    got = wire_unpack_host(yc[cols].cpu().numpy(), ctx.wire_widths(12), 12, ctx.n)
    del xc, yc
    torch.cuda.empty_cache()
    assert (got == o.pcmm_a(x, W, cols=cols, nthreads=NTH)).all()


@pytest.mark.parametrize("d,m", [(1536, 1536), (4096, 1536)])
def test_compact_paper_table3_shapes_n14(torch_cuda, d, m):
    """Two of the paper's Table III PCMM shapes at its default ring N' = 2^14, l = 12 (bench.py paper_table3_n14 on the
    compact layout): Q/K/V 1536x1536 and down 4096->1536, sampled columns == the oracle."""
    from paper_2509_09424_b200 import Context
    torch = torch_cuda
    ctx = Context(14, 12, 4, 3)
    o = oracle.Oracle(14, 12, 4, 3)
    x = synth.gen_words(15000 + d, o.q, d, 12, o.n)
    W = synth.gen_W(15001 + m, d, m)
    from paper_2509_09424_b200.ensi import wire_unpack_host
    xc = _compact_dev(torch, ctx, x, 12)
    yc = torch.empty((m, ctx.wire_bytes(12)), dtype=torch.uint8, device="cuda")
    ctx.pcmm_ternary_compact(xc, ctx.weights(W), yc, level=12)
    torch.cuda.synchronize()
    cols = [0, 777, m - 1]
    got = wire_unpack_host(yc[cols].cpu().numpy(), ctx.wire_widths(12), 12, ctx.n)
    assert (got == o.pcmm_a(x, W, cols=cols, nthreads=NTH)).all()
